#!/bin/bash
# Copy gpurun_out/ev (tools/final_evidence.sh) into profiles/ and print the table.
set -e
cd "$(dirname "$0")/.."
for f in gpurun_out/ev/bench_*.json; do b=$(basename $f .json); tail -1 $f > profiles/r01_final_$b.json; done
cp gpurun_out/ev/launches_c2.csv profiles/r01_final_launches_c2_cpinn.csv
cp gpurun_out/ev/pytest_gpu.txt profiles/r01_final_pytest_gpu.txt
cp gpurun_out/ev/smoke.txt profiles/r01_final_smoke.txt
rm -f profiles/k1_dram_bytes.json
python tools/dram_table.py "C2-poisson-4x4-6x40 cpinn" gpurun_out/ev/k1_c2.ncu-rep "C3-burgers-xpinn-4x2-5x20 xpinn" \
    gpurun_out/ev/k1_c3.ncu-rep "C4-ns-xpinn-4x2-5x80 xpinn" gpurun_out/ev/k1_c4.ncu-rep \
    "C5-heatinv-xpinn-voronoi10-3x80 xpinn" gpurun_out/ev/k1_c5.ncu-rep > /dev/null
for w in c2 c3 c4 c5; do
  python tools/ncu_summary.py gpurun_out/ev/k1_$w.ncu-rep profiles/r01_final_k1_${w}_ncu_summary.json > /dev/null
done
for f in profiles/r01_final_bench_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
r = d.get("roofline") or {}
c = d.get("cpu_baseline") or {}
print(sys.argv[1].split("/")[-1], d["config"]["workload"], "%.4g" % d["value"], round(d["ms_per_step"], 4),
      round(r.get("frac") or 0, 4), r.get("k1_ms_per_launch"), r.get("traffic"), "e2e %.4g" % d["e2e"]["value"],
      c.get("value"), c.get("cores"), d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
PY
done
