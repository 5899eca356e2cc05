#!/bin/bash
# bench each libvar_*.so (PINN_DD_LIB) against the default library on the given workloads
mkdir -p gpurun_out/var
for w in ${WORKLOADS:-c2 c4}; do
  st=""; [ "$w" = c4 ] && st="--steps 30"
  for f in paper_2104_10013_b200/libpinn_dd.so paper_2104_10013_b200/libvar_*.so; do
    n=$(basename $f .so)
    PINN_DD_LIB=$PWD/$f python bench.py --no-cpu --workload $w $st > gpurun_out/var/${w}_$n.json 2>&1
    tail -1 gpurun_out/var/${w}_$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $n', round(d['roofline']['k1_ms_per_launch'],4), round(d['roofline']['frac'],4))"
  done
done
