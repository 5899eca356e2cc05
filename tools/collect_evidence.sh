#!/bin/bash
# Copy gpurun_out/ev (tools/final_evidence.sh) into profiles/ with a round tag
# and print the table.  usage: collect_evidence.sh r02
set -e
cd "$(dirname "$0")/.."
R=${1:-r02}
for f in gpurun_out/ev/bench_*.json; do b=$(basename $f .json); tail -1 $f > profiles/${R}_$b.json; done
[ -f gpurun_out/ev/launches_c4.csv ] && cp gpurun_out/ev/launches_c4.csv profiles/${R}_launches_c4.csv
[ -f gpurun_out/ev/pytest_gpu.txt ] && cp gpurun_out/ev/pytest_gpu.txt profiles/${R}_pytest_gpu.txt
[ -f gpurun_out/ev/smoke.txt ] && cp gpurun_out/ev/smoke.txt profiles/${R}_smoke.txt
for f in profiles/${R}_bench_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read())
except Exception as e:
    print(sys.argv[1], "unparsable", e); sys.exit(0)
r = d.get("roofline") or {}
c = d.get("cpu_baseline") or {}
print(sys.argv[1].split("/")[-1], d["config"]["workload"], "%.4g" % d["value"], round(d["ms_per_step"], 4),
      round(r.get("frac") or 0, 4), r.get("k1_ms_per_launch"), r.get("traffic"), "e2e %.4g" % d["e2e"]["value"],
      c.get("value"), c.get("cores"), d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
PY
done
