#!/bin/bash
# one ncu --set full capture of K1 per workload (development tool; run on the GPU box)
# usage: tools/ncu_k1.sh WORKLOAD[_tf32]...   -> gpurun_out/ev/k1_<w>.ncu-rep
set -u
O=gpurun_out/ev
mkdir -p $O
for w in "$@"; do
  extra=""; K='regex:k_fused<'
  case $w in *_tf32) extra="--tf32"; K='regex:k_fused_tc<';; esac
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -c 1 \
      -o $O/k1_$w python bench.py --no-cpu --workload ${w%_tf32} $extra --steps 2 --warmup 3 > /dev/null 2>&1
done
ls -la $O
