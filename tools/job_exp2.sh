#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
for v in "NSF_LPT=0" "NSF_LPT=1"; do
  echo "== stats $v"; env $v NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/stats.so python tools/stats_run.py C3 250 32 2>&1 | tail -1
done
for c in C3 C2; do for rep in 1 2; do
for v in "NSF_LPT=0" "NSF_LPT=1"; do
  echo -n "$c [$v] "; env $v python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})"
done; done; done
