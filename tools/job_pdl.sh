cd "${GRAFT_REPO_ROOT}"
for c in C3 C2; do for rep in 1 2; do for v in 0 1; do echo -n "$c PDL=$v "; NSF_PDL=$v NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/pdl.so python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/pdl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
