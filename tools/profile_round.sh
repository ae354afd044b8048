#!/bin/bash
# One GPU call's worth of evidence for a config (run under gpurun):
#   bench line, ncu launch list of a short bench, ncu --set full of the top kernel.
#   CONFIG=C3 KERNEL=k_g2p2g TAG=r1 bash tools/profile_round.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CONFIG=${CONFIG:-C3}; KERNEL=${KERNEL:-k_g2p2g}; TAG=${TAG:-r1}
CMD="python bench.py --config $CONFIG --steps 20 --warmup 3 --no-cpu-baseline --e2e-iters 1"
python bench.py --config $CONFIG ${BENCH_ARGS} > gpurun_out/bench_${TAG}_${CONFIG}.json 2> gpurun_out/bench_${TAG}_${CONFIG}.err || exit 1
[ -n "$NO_NCU" ] && exit 0
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${CONFIG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s 6 -c 2 \
    -o gpurun_out/prof_${TAG}_${CONFIG} $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
