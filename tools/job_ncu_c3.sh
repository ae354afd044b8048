#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
CMD="python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-iters 1"
$CMD > gpurun_out/c3_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_g2p2g|k_grid_update_list" -s 30 -c 2 -o gpurun_out/prof_c3_head $CMD > gpurun_out/ncu_c3.log 2>&1
ncu -i gpurun_out/prof_c3_head.ncu-rep --page source --csv -k regex:k_g2p2g --print-source sass > gpurun_out/sass_c3_head.csv 2>/dev/null
ncu -i gpurun_out/prof_c3_head.ncu-rep --page raw --csv > gpurun_out/raw_c3_head.csv 2>/dev/null
