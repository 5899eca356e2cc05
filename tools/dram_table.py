"""Write profiles/k1_dram_bytes.json: DRAM bytes per K1 launch per bench workload,
from one ncu --set full capture each.
usage: python tools/dram_table.py "WORKLOAD KEY" report.ncu-rep [...pairs]"""
import csv, io, json, os, subprocess, sys

out_path = os.path.join(os.path.dirname(__file__), "..", "profiles", "k1_dram_bytes.json")
table = json.load(open(out_path)) if os.path.exists(out_path) else {}
table = {k: v for k, v in table.items() if isinstance(v, dict)}
args = sys.argv[1:]
for key, rep in zip(args[::2], args[1::2]):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    d = {k: float(x) * scale[un] for k, un, x in zip(h, u, v) if k in ("dram__bytes_read.sum", "dram__bytes_write.sum")}
    table[key] = {"dram_bytes_per_launch": int(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]),
                  "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "",
                  "source": os.path.basename(rep) + " (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full)"}
json.dump(table, open(out_path, "w"), indent=1)
print(json.dumps(table, indent=1))
