#!/bin/bash
# A/B compile-time knobs on the GPU box: bash tools/ab_defines.sh "A=1" "A=0 B=2" ...
# (each argument is one NSF_DEFINES set; the library is rebuilt per set)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for d in "$@"; do
  NSF_DEFINES="$d" python -m paper_2310_17790_b200.build > gpurun_out/ab_build.log 2>&1 || { cat gpurun_out/ab_build.log; exit 1; }
  for i in 1 2; do echo "[$d]"; python bench.py --no-cpu-baseline --e2e-iters 1 ${BENCH_ARGS} 2>&1 | tail -1 | cut -c1-220; done
done
python -m paper_2310_17790_b200.build > /dev/null 2>&1
