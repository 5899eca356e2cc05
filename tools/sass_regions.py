"""Split an ncu SASS source page (csv) into straight-line segments and report
per-segment instruction and stall-sample shares (development tool).
usage: python tools/sass_regions.py sass.csv [min_share]"""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
src = [r[ix["Source"]].strip() for r in data]
E = [int(r[ix["Instructions Executed"]] or 0) for r in data]
S = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
TE, TS = sum(E), sum(S)
segs = []
b = 0
for i in range(1, len(data) + 1):
    if i == len(data) or E[i] != E[b]:
        segs.append((b, i))
        b = i
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
print(f"total inst {TE:.3e} samples {TS}")
for b, e in segs:
    s = sum(S[b:e]); ex = sum(E[b:e])
    if s / TS < mn:
        continue
    rs = collections.Counter()
    for i in range(b, e):
        for h in reasons:
            rs[h] += int(data[i][ix[h]] or 0)
    ops = collections.Counter(src[i].split()[0 if not src[i].startswith('@') else 1].split('.')[0] for i in range(b, e))
    top = ", ".join(f"{k[6:]}={v / max(1, s):.2f}" for k, v in rs.most_common(6))
    print(f"[{b:5d},{e:5d}) x{E[b]:>9d} inst {ex / TE * 100:5.1f}% samp {s / TS * 100:5.1f}% | {top}")
    print("      ops:", dict(ops.most_common(8)))
