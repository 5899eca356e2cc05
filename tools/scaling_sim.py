"""Per-GPU compute of the multi-GPU placements, measured on ONE GPU (no NCCL:
the remote payload rows stay at their last values).  For N in 1, 2, 4, 8 the
handle of rank 0 under bench.py's placement runs K graph-free iterations of
K2 -> K1 interior -> K1 interface + K5 (the phased calls); reports ms per
iteration, the implied strong / weak efficiency of the COMPUTE part and the
chunk count.  usage: python tools/scaling_sim.py [c4|c2|c3|c5] [--tf32]"""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD, FLAG_TF32

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
fl = FLAG_TF32 if "--tf32" in sys.argv else 0
res = {}
for n in (1, 2, 4, 8):
    prob, owner, scaling = bench.workload(wl, "cpinn" if wl == "c2" else "xpinn", n)
    local = [q for q in range(prob.n_sub) if owner[q] == 0]
    h = PinnDD(prob, local, owner, 0, device="cuda:0", flags=fl)
    K = 30 if wl == "c4" else 200
    def it():
        h.interface_payload()
        h.lib.pinn_dd_loss_grad_interior(h.h)
        h.lib.pinn_dd_loss_grad_interface(h.h, None, None)
        h.adam()
    for _ in range(5):
        it()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        it()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[n] = ms
    info = h.plan_info()
    base = res[1]
    eff = base / ms / n if scaling == "strong" else base / ms
    print(json.dumps(dict(workload=prob.name, n_gpus=n, local_subdomains=len(local), points=h.n_points,
                          ms_per_iter=ms, chunks=info[2], grid=info[3], compute_efficiency=eff, scaling=scaling,
                          tf32=bool(fl))), flush=True)
    h.close()
