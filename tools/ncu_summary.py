"""Summarise an ncu report: key throughput metrics, stall reasons, hot source lines."""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v)); un = dict(zip(h, u))
keys = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'smsp__inst_executed.sum']
out = {k: [d.get(k), un.get(k)] for k in keys}
for k in h:
    if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
        if float(d[k] or 0) > 0.01:
            out[k.replace('smsp__average_warps_issue_stalled_', 'stall_').replace('_per_issue_active.ratio', '')] = [d[k], '']
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], 'w'), indent=1)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; agg = {}; hdr = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == 'File Path':
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = r; continue
    if hdr and r and r[0].isdigit():
        try:
            s = int(r[hdr.index('Warp Stall Sampling (All Samples)')]); n = int(r[hdr.index('Instructions Executed')])
        except Exception:
            continue
        agg[(cur, int(r[0]))] = (s, n, r[1].strip()[:80])
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{k[0][:14]:14s}{k[1]:5d} {100*v[0]/tot:5.1f}% {100*v[1]/toti:5.1f}%i  {v[2]}")
