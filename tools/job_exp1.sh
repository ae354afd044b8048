#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
export NSF_MPM_LIB_STATS="$PWD/paper_2310_17790_b200/_ab/stats.so"
for v in default barrier; do
  if [ $v = barrier ]; then export NSF_FUSED_GU=barrier; else unset NSF_FUSED_GU; fi
  echo "== stats $v"; NSF_MPM_LIB=$NSF_MPM_LIB_STATS python tools/stats_run.py C3 250 32 2>&1 | tail -3
done
unset NSF_FUSED_GU
for rep in 1 2; do
for v in "" "NSF_FUSED_GU=barrier" "NSF_FUSED_VARIANT=dense2"; do
  echo -n "C3 [$v] "; env $v python bench.py --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})"
done; done
