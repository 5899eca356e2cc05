#!/bin/bash
# Round-end evidence: bench lines for every workload/method, the oracle arm,
# the ncu launch list of the default bench command and one full K1 capture.
set -u
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench_c2_cpinn.json 2> gpurun_out/ev/bench_c2_cpinn.err
python bench.py --method xpinn --no-cpu > gpurun_out/ev/bench_c2_xpinn.json 2>&1
python bench.py --method hybrid --no-cpu > gpurun_out/ev/bench_c2_hybrid.json 2>&1
python bench.py --method dp --no-cpu > gpurun_out/ev/bench_c2_dp.json 2>&1
python bench.py --workload c3 > gpurun_out/ev/bench_c3.json 2>&1
python bench.py --workload c4 --steps 30 > gpurun_out/ev/bench_c4.json 2>&1
python bench.py --workload c5 > gpurun_out/ev/bench_c5.json 2>&1
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ev/bench_reference_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c2.csv \
    python bench.py --no-cpu --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"k_fused<.*\(int\)0, \(int\)0>" -c 1 -o gpurun_out/ev/k1_c2 \
    python bench.py --no-cpu --steps 2 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out/ev
