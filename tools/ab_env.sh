cd "${GRAFT_REPO_ROOT}"
for cfg in C3 C5; do for rep in 1 2; do for m in block 1; do
  echo "== $cfg NSF_REORDER_CELLS=$m"
  NSF_REORDER_CELLS=$m python tools/trace_steps.py --config $cfg 2>&1 | head -2 | tail -1
  NSF_REORDER_CELLS=$m python bench.py --config $cfg --no-cpu-baseline --e2e-iters 1 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*'
done; done; done
