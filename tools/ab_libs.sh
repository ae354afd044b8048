#!/bin/bash
# Same-box A/B of prebuilt library variants (run under gpurun):
#   bash tools/ab_libs.sh _ab/base.so _ab/new.so      (paths relative to the package dir)
# Each variant runs tools/trace_steps.py and a short bench, interleaved twice.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
  for l in "$@"; do
    echo "== $l"
    NSF_MPM_LIB="$PWD/paper_2310_17790_b200/$l" python tools/trace_steps.py ${TRACE_ARGS} 2>&1 | head -2
    NSF_MPM_LIB="$PWD/paper_2310_17790_b200/$l" python bench.py --no-cpu-baseline --e2e-iters 1 ${BENCH_ARGS} 2>&1 | tail -1 | cut -c100-190
  done
done
