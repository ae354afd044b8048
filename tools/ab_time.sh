#!/bin/bash
# Same-box A/B of prebuilt library variants on substep time (run under gpurun):
#   CONFIGS="C3 C2" bash tools/ab_time.sh _ab/base.so _ab/new.so   (paths relative to the package dir)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for c in ${CONFIGS:-C3}; do
  for rep in 1 2; do
    for l in "$@"; do
      echo -n "$l: "
      NSF_MPM_LIB="$PWD/paper_2310_17790_b200/$l" python tools/align_probe.py --config $c --shifts 0,0,0 --steps ${STEPS:-100} 2>&1 | tail -1
    done
  done
done
