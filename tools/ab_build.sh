#!/bin/bash
# Build library variants here (no GPU needed) into paper_2310_17790_b200/_ab/<name>.so:
#   bash tools/ab_build.sh "base:" "nof2:NSF_F2_G2P=0 NSF_F2_P2G=0" ...
# then time them on the box with tools/ab_run.sh base nof2 ...
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2310_17790_b200/_ab
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  NSF_DEFINES="$defs" python -m paper_2310_17790_b200.build > /dev/null
  cp paper_2310_17790_b200/libnsf_mpm.so "paper_2310_17790_b200/_ab/$name.so"
  echo "built $name [$defs]"
done
python -m paper_2310_17790_b200.build > /dev/null
