cd "${GRAFT_REPO_ROOT}"
timeout 900 python -m pytest tests/test_gpu_far.py tests/test_gpu_edge_cases.py tests/test_gpu_checked.py -x -q 2>&1 | tail -3
for c in C3 C4; do for rep in 1 2; do for v in kernel pro; do echo -n "$c [$v] "; NSF_FUSED_GU=$v python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
for v in kernel pro; do echo -n "C3 w20 [$v] "; NSF_FUSED_GU=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us')"
done
