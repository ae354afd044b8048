#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
export NSF_FUSED_GU=flow
for c in C3; do
for v in fnofence ffenceonly fnoarr; do
  echo -n "$c [$v] "; NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/$v.so python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done
