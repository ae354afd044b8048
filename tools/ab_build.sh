#!/bin/bash
# Build library variants here (no GPU needed) into paper_2310_17790_b200/_ab/<name>.so, in parallel
# (each in its own build directory):
#   bash tools/ab_build.sh "base:" "nof2:NSF_F2_G2P=0 NSF_F2_P2G=0" ...
# then time them on the box with tools/ab_run.sh base nof2 ...
cd "$(dirname "$0")/.."
mkdir -p paper_2310_17790_b200/_ab
pids=()
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  ( NSF_DEFINES="$defs" NSF_BUILD_DIR="$PWD/paper_2310_17790_b200/_ab/_build_$name" \
    NSF_LIB_OUT="$PWD/paper_2310_17790_b200/_ab/$name.so" python -m paper_2310_17790_b200.build > /dev/null \
    && echo "built $name [$defs]" || echo "FAILED $name" ) &
  pids+=($!)
done
wait "${pids[@]}"
