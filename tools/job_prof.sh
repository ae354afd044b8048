#!/bin/bash
# final evidence of the round (bench lines, launch lists, ncu summaries) -> gpurun_out/*r2f*
cd "${GRAFT_REPO_ROOT}"
TAG=r2f
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_C3_driver.json 2> gpurun_out/bench_${TAG}_C3_driver.err || exit 1
python bench.py --config C3 --preroll 70 --warmup 5 --steps 424 --no-cpu-baseline > gpurun_out/bench_${TAG}_C3_run.json 2> gpurun_out/bench_${TAG}_C3_run.err
for c in C1 C2 C4 C5; do
  python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
python bench.py --config C3 --steps 64 --warmup 5 --no-cpu-baseline --deterministic > gpurun_out/bench_${TAG}_C3_det.json 2> gpurun_out/bench_${TAG}_C3_det.err
for f in C3_driver C3_run C1 C2 C4 C5 C3_det; do python - $f gpurun_out/bench_${TAG}_$f.json <<'PY'
import json,sys
for l in open(sys.argv[2]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['ms_per_step']*1e3,2), 'us', round(d.get('hbm_alg_frac_whole_step',0),4), 'b2b', round(d['back_to_back']['ms_per_step']*1e3,2), {k: round(x*1e3,1) for k,x in d['kernel_ms_per_substep'].items()})
PY
done
for c in C3 C5; do
  CMD="python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-iters 1"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$c.csv $CMD > /dev/null 2>&1
done
C3CMD="python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-iters 1"
# -s 620: past the 250-substep pre-roll (2 launches per substep + 7 re-binnings), i.e. mid-run kernels
ncu --set full --clock-control none --import-source on -k "regex:k_g2p2g|k_grid_update_list" -s 620 -c 6 -o gpurun_out/prof_${TAG}_C3 $C3CMD > gpurun_out/ncu_full3.log 2>&1
ncu --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum.per_second,lts__t_sectors.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_g2p2g -s 310 -c 2 --csv --log-file gpurun_out/red_${TAG}_C3.csv $C3CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_nsf_mlp_tc|k_g2p_nsf" -s 6 -c 2 -o gpurun_out/prof_${TAG}_C5 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1 > gpurun_out/ncu_full5.log 2>&1
for c in C3 C5; do
  [ -f gpurun_out/prof_${TAG}_$c.ncu-rep ] && python tools/summarize_ncu.py gpurun_out/prof_${TAG}_$c.ncu-rep gpurun_out/ncu_${TAG}_$c.txt
done
rm -f gpurun_out/*.ncu-rep
echo "profile rc=$?"
