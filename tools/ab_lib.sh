#!/bin/bash
# A/B alternative library builds on the GPU box (development tool):
# tools/ab_lib.sh "vA vB ..." WORKLOAD...  -> each paper_2104_10013_b200/libpinn_dd_<v>.so swapped in turn
set -u
L=paper_2104_10013_b200
cp $L/libpinn_dd.so /tmp/libpinn_dd_real.so
for v in $1; do
  cp $L/libpinn_dd_$v.so $L/libpinn_dd.so
  shift 0
  bash tools/ab_quick.sh $v "${@:2}"
done
cp /tmp/libpinn_dd_real.so $L/libpinn_dd.so
