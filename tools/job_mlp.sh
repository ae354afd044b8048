#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
timeout 900 python -m pytest tests/test_gpu_nsf.py tests/test_gpu_inference.py -x -q 2>&1 | tail -4
for rep in 1 2; do for v in 0 1; do echo -n "C5 MLP_WS=$v "; NSF_MLP_WS=$v python bench.py --config C5 --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()}, d['roofline']['frac'])
    elif 'rror' in l: print(l.strip()[:300])"
done; done
