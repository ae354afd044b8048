#!/bin/bash
# Round evidence (run under gpurun): bench lines for every config, then the ncu
# launch list + a full capture of the top kernel(s) for C3 and C5.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
for c in C1 C2 C4 C5; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err || exit 1
done
python bench.py > gpurun_out/bench_${TAG}_C3.json 2> gpurun_out/bench_${TAG}_C3.err || exit 1
[ -n "$NO_NCU" ] && exit 0
C3CMD="python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1"
C5CMD="python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1"
$C3CMD > gpurun_out/plain3.log 2>&1 && $C5CMD > gpurun_out/plain5.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_C3.csv $C3CMD > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_C5.csv $C5CMD > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_g2p2g -s 6 -c 1 -o gpurun_out/prof_${TAG}_C3 $C3CMD > gpurun_out/ncu_full3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:k_nsf_mlp_tc|k_g2p_nsf" -s 6 -c 2 -o gpurun_out/prof_${TAG}_C5 $C5CMD > gpurun_out/ncu_full5.log 2>&1
echo "profile rc=$?"
