#!/bin/bash
# Same-box A/B of prebuilt libraries (run under gpurun):
#   CONFIGS="C3 C2" REPS=2 STEPS=64 bash tools/job_ab.sh base scan ...   (paper_2310_17790_b200/_ab/<name>.so)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for c in ${CONFIGS:-C3}; do for rep in $(seq ${REPS:-2}); do
for v in "$@"; do
  echo -n "$c [$v] "; NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/$v.so python bench.py --config $c --steps ${STEPS:-64} --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
