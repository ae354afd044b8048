#!/bin/bash
# Build the committed HEAD and the working tree into paper_2310_17790_b200/_ab/{base,new}.so
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2310_17790_b200/_ab
git stash -q
trap 'git stash pop -q' EXIT
python -m paper_2310_17790_b200.build > /dev/null
cp paper_2310_17790_b200/libnsf_mpm.so paper_2310_17790_b200/_ab/base.so
git stash pop -q
trap - EXIT
python -m paper_2310_17790_b200.build > /dev/null
cp paper_2310_17790_b200/libnsf_mpm.so paper_2310_17790_b200/_ab/new.so
ls -la paper_2310_17790_b200/_ab
