#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
export NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/stats.so
for pre in 257 265 273 281; do python tools/stats_run.py C3 $pre 6 2>&1 | tail -3; done
