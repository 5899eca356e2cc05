#!/bin/bash
# Round-end evidence: bench lines for every workload/method, the oracle arm,
# the ncu launch list of the default bench command and one full K1 capture per
# workload (DRAM bytes -> profiles/k1_dram_bytes.json via tools/dram_table.py).
# usage: final_evidence.sh [bench|tests|ncu WORKLOADS...]  (gpurun returns <= 64 MiB
# per call: one full K1 report is ~22 MB, so the captures go in separate calls)
set -u
O=gpurun_out/ev
mkdir -p $O
case "${1:-bench}" in
ncu)
  shift
  K='k_fused<.*\(int\)2, \(int\)(256|128)>'
  for w in "$@"; do
    ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k regex:"$K" -c 1 -o $O/k1_$w python bench.py --no-cpu --workload $w --steps 2 --warmup 3 > /dev/null 2>&1
  done
  ls -la $O
  ;;
tests)
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
  tail -3 $O/pytest_gpu.txt
  ;;
bench)
  python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
  python bench.py --workload c2 > $O/bench_c2_cpinn.json 2>&1
  python bench.py --workload c2 --method xpinn --no-cpu > $O/bench_c2_xpinn.json 2>&1
  python bench.py --workload c2 --method hybrid --no-cpu > $O/bench_c2_hybrid.json 2>&1
  python bench.py --workload c2 --method dp --no-cpu > $O/bench_c2_dp.json 2>&1
  python bench.py --workload c3 > $O/bench_c3.json 2>&1
  python bench.py --workload c3x8 --no-cpu > $O/bench_c3x8.json 2>&1
  python bench.py --tf32 --no-cpu > $O/bench_c4_tf32.json 2>&1
  python bench.py --workload c5 --tf32 --no-cpu > $O/bench_c5_tf32.json 2>&1
  python bench.py --workload c5 > $O/bench_c5.json 2>&1
  python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_c4.json 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
      python bench.py --no-cpu --steps 2 --warmup 3 > /dev/null 2>&1
  ls -la $O
  ;;
esac
