#!/bin/bash
# final check of the round: smoke, GPU tests, the driver's bench line and the reference arm
cd "${GRAFT_REPO_ROOT}"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_C3.json 2> gpurun_out/final_C3.err; tail -c 600 gpurun_out/final_C3.json
python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 2>/dev/null | tail -1 | cut -c1-400
python bench.py > gpurun_out/final_default.json 2> gpurun_out/final_default.err; python - <<'PY'
import json
for f in ['gpurun_out/final_C3.json','gpurun_out/final_default.json']:
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(f, d['steps'], round(d['ms_per_step']*1e3,2), 'us', round(d['hbm_alg_frac_whole_step'],4), 'b2b', round(d['back_to_back']['ms_per_step']*1e3,2), 'launches', d['gpu_launches'])
PY
