#!/bin/bash
# Round-2 evidence (run under gpurun): bench lines for every config (C3 twice: the
# driver's --steps 20 --warmup 5 window and the whole 500-substep run), ncu launch
# lists (C3, C4, C5), full captures of the top kernels of every config plus the
# grid-update and re-binning kernels, and the L2 reduction counters of the fused P2G.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2}
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_C3_driver.json 2> gpurun_out/bench_${TAG}_C3_driver.err || exit 1
python bench.py --config C3 --preroll 0 --warmup 3 --steps 496 --no-cpu-baseline > gpurun_out/bench_${TAG}_C3_full.json 2> gpurun_out/bench_${TAG}_C3_full.err || exit 1
for c in C1 C2 C4 C5; do
  python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err || exit 1
done
python bench.py --config C3 --steps 64 --warmup 5 --no-cpu-baseline --deterministic > gpurun_out/bench_${TAG}_C3_det.json 2> gpurun_out/bench_${TAG}_C3_det.err
[ -n "$NO_NCU" ] && exit 0
for c in C3 C4 C5; do
  CMD="python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-iters 1"
  $CMD > gpurun_out/plain_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$c.csv $CMD > /dev/null 2>&1
done
C3CMD="python bench.py --config C3 --steps 40 --warmup 5 --no-cpu-baseline --e2e-iters 1"
ncu --set full --clock-control none --import-source on -k "regex:k_g2p2g|k_grid_update_list|k_keys_hist|k_scan|k_copy_cells|k_cell|k_halo|k_lpt" -s 40 -c 9 -o gpurun_out/prof_${TAG}_C3 $C3CMD > gpurun_out/ncu_full3.log 2>&1
ncu --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum.per_second,lts__t_sectors.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_g2p2g -s 6 -c 2 --csv --log-file gpurun_out/red_${TAG}_C3.csv $C3CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_g2p2g -s 4 -c 1 -o gpurun_out/prof_${TAG}_C4 python bench.py --config C4 --steps 8 --warmup 3 --no-cpu-baseline --e2e-iters 1 > gpurun_out/ncu_full4.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_nsf_mlp_tc|k_g2p_nsf" -s 6 -c 2 -o gpurun_out/prof_${TAG}_C5 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1 > gpurun_out/ncu_full5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_g2p2g -s 6 -c 1 -o gpurun_out/prof_${TAG}_C2 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1 > gpurun_out/ncu_full2.log 2>&1
for c in C3 C2 C4; do
  ncu -i gpurun_out/prof_${TAG}_$c.ncu-rep --page source --csv -k regex:k_g2p2g --print-source sass > gpurun_out/sass_${TAG}_$c.csv 2>/dev/null
done
# summaries on the box (the reports exceed the 64 MiB copy-back): text + SASS attribution only
for c in C3 C2 C4 C5; do
  [ -f gpurun_out/prof_${TAG}_$c.ncu-rep ] && python tools/summarize_ncu.py gpurun_out/prof_${TAG}_$c.ncu-rep gpurun_out/ncu_${TAG}_$c.txt
done
for c in C3 C2 C4; do
  o=paper_2310_17790_b200/_build/kernels_tiled.cu.o
  python tools/sass_lines.py gpurun_out/sass_${TAG}_$c.csv $o k_g2p2g 40 > gpurun_out/sass_lines_${TAG}_$c.txt 2>&1
  gzip -f gpurun_out/sass_${TAG}_$c.csv
done
rm -f gpurun_out/*.ncu-rep
echo "profile rc=$?"
