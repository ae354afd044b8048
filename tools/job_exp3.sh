#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
timeout 900 python -m pytest tests/test_gpu_flow.py tests/test_gpu_edge_cases.py -x -q 2>&1 | tail -15
for c in C3 C2 C4; do for rep in 1 2; do
for v in "NSF_FUSED_GU=kernel" "NSF_FUSED_GU=flow"; do
  echo -n "$c [$v] "; env $v python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
