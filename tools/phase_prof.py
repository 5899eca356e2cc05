"""Per-phase cycle split of the fused K1 launch (development tool).  Needs the
library built with -DPINN_PHASE_PROF (tools/phase_prof.sh swaps it in): CTAs
0..3 print the clock cycles thread 0 spent per phase; this script runs two
graph-free steps of a bench workload and prints the second step's split.
usage: python tools/phase_prof.py WORKLOAD [--tf32]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2104_10013_b200.binding import PinnDD, FLAG_TF32

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
fl = FLAG_TF32 if "--tf32" in sys.argv else 0
prob, owner, scaling = bench.workload(wl, "cpinn" if wl == "c2" else "xpinn", 1)
local = [q for q in range(prob.n_sub) if owner[q] == 0]
h = PinnDD(prob, local, owner, 0, device="cuda:0", flags=fl)
h.step(1, want_loss=False)
torch.cuda.synchronize()
print("---MARK---", wl, flush=True)
h.step(1, want_loss=False)
torch.cuda.synchronize()
h.close()
