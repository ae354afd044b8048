#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/x5_C3.json 2> gpurun_out/x5_C3.err
python - <<'PY'
import json
for l in open('gpurun_out/x5_C3.json'):
    if l.startswith('{'):
        d=json.loads(l); print('C3 driver', round(d['ms_per_step']*1e3,2), 'us; back-to-back', round(d['back_to_back']['ms_per_step']*1e3,2), d['back_to_back']['hbm_alg_frac_whole_step'], 'e2e', d['e2e']['value'])
PY
tail -3 gpurun_out/x5_C3.err
python tools/warm_time.py C3 250 64 3
NSF_WRITE_EVERY=1 python tools/warm_time.py C3 250 64 3
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
