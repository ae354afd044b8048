#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/flow2.so timeout 600 python -m pytest tests/test_gpu_flow.py -x -q 2>&1 | tail -3
NSF_FUSED_GU=flow NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/stats.so python tools/stats_run.py C3 250 32 2>&1 | tail -3
for c in C3 C2; do for rep in 1 2; do
for v in "NSF_FUSED_GU=kernel" "NSF_FUSED_GU=flow"; do
  echo -n "$c [$v] "; env $v NSF_MPM_LIB=$PWD/paper_2310_17790_b200/_ab/flow2.so python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us', {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
    elif 'rror' in l: print(l.strip()[:300])"
done; done; done
