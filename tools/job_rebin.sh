#!/bin/bash
# re-binning period A/B on C3: flushed 96-substep windows (a whole number of periods for 16, 24, 32, 48) and back to back
cd "${GRAFT_REPO_ROOT}"
for r in 16 24 32 48; do
  for rep in 1 2; do
    echo -n "rebin_every $r: "; NSF_REBIN_EVERY=$r python bench.py --config C3 --steps 96 --warmup 5 --no-cpu-baseline --e2e-iters 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step']*1e3,2), 'us flushed;', 'rebins', d['config']['window']['rebins_in_window'], '; b2b', round(d['back_to_back']['ms_per_step']*1e3,2), d['back_to_back']['substeps'])"
  done
done
