#!/bin/bash
# GPU tests + one bench line per config (run under gpurun); TAG names the output files
cd "${GRAFT_REPO_ROOT}"
T=${TAG:-x}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; tail -3 gpurun_out/${T}_tests.log
for c in ${CONFIGS:-C3 C2 C4 C5 C1}; do
  python bench.py --config $c ${BENCH_ARGS} > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  python - "$c" gpurun_out/${T}_bench_$c.json <<'PY'
import json,sys
for l in open(sys.argv[2]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['ms_per_step']*1e3,2), 'us', d.get('hbm_alg_frac_whole_step'), {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
PY
done
