cd "${GRAFT_REPO_ROOT}"
for c in C4 C3; do for v in 0 1; do echo -n "$c LPT=$v "; NSF_LPT=$v python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})"
done; done
