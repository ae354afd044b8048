#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
export NSF_MLP_WS=0
NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/mlp_pair.so timeout 900 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_inference.py -x -q 2>&1 | tail -2
CONFIGS=C5 bash tools/job_ab.sh mlp_scalar mlp_pair
