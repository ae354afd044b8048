#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
CMD="python bench.py --config C5 --steps 6 --warmup 3 --preroll 4 --no-cpu-baseline --e2e-iters 1"
NSF_MLP_WS=1 ncu --set full --clock-control none --import-source on -k "regex:k_nsf_mlp" -s 4 -c 1 -o gpurun_out/prof_mlp_ws $CMD > gpurun_out/ncu_mlp_ws.log 2>&1
NSF_MLP_WS=0 ncu --set full --clock-control none --import-source on -k "regex:k_nsf_mlp" -s 4 -c 1 -o gpurun_out/prof_mlp_tc $CMD > gpurun_out/ncu_mlp_tc.log 2>&1
for v in ws tc; do
  ncu -i gpurun_out/prof_mlp_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_mlp_$v.csv 2>/dev/null
  ncu -i gpurun_out/prof_mlp_$v.ncu-rep --page raw --csv > gpurun_out/raw_mlp_$v.csv 2>/dev/null
done
ls -la gpurun_out/ | tail
