#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
L=$PWD/paper_2310_17790_b200/_ab
CONFIGS="C3" REPS=2 STEPS=64 bash tools/job_ab.sh base tw
python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/x9_C3.json 2> gpurun_out/x9_C3.err
python - <<'PY'
import json
for l in open('gpurun_out/x9_C3.json'):
    if l.startswith('{'):
        d=json.loads(l); print('C3 driver', round(d['ms_per_step']*1e3,2), 'us; back-to-back', round(d['back_to_back']['ms_per_step']*1e3,2), d['back_to_back']['hbm_alg_frac_whole_step'], 'e2e', d['e2e']['value'])
PY
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
