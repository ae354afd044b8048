#!/bin/bash
# re-entry baseline: GPU tests, C3 driver-window and whole-run bench lines, C5 line
cd "${GRAFT_REPO_ROOT}"
T=${TAG:-base}
python bench.py --config C3 --steps 20 --warmup 5 > gpurun_out/${T}_C3_driver.json 2> gpurun_out/${T}_C3_driver.err
python bench.py --config C3 --steps 496 --warmup 6 --preroll 0 --no-cpu-baseline --e2e-iters 1 > gpurun_out/${T}_C3_full.json 2> gpurun_out/${T}_C3_full.err
python bench.py --config C5 --no-cpu-baseline --e2e-iters 1 > gpurun_out/${T}_C5.json 2> gpurun_out/${T}_C5.err
for f in C3_driver C3_full C5; do python - $f gpurun_out/${T}_$f.json <<'PY'
import json,sys
for l in open(sys.argv[2]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['ms_per_step']*1e3,2), 'us', d.get('hbm_alg_frac_whole_step'), {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
PY
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; tail -3 gpurun_out/${T}_tests.log
