#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in 20 64; do for rep in 1 2; do for v in 0 1; do echo -n "C3 w$w DEFER=$v "; NSF_DEFERRED_REORDER=$v python bench.py --steps $w --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
for c in C2 C4; do for v in 0 1; do echo -n "$c DEFER=$v "; NSF_DEFERRED_REORDER=$v python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})"
done; done
