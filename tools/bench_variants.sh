#!/bin/bash
# bench each libvar_*.so (PINN_DD_LIB) against the default library
python bench.py --no-cpu --steps 100 > gpurun_out/var_default.log 2>&1
for f in paper_2104_10013_b200/libvar_*.so; do
  n=$(basename $f .so)
  PINN_DD_LIB=$PWD/$f python bench.py --no-cpu --steps 100 > gpurun_out/$n.log 2>&1
done
