"""Per-GPU step time of the multi-GPU placements on ONE GPU, through the real
graph-replayed pinn_dd_step with the peer-store transport: rank 0's
subdomains under bench.py's placement, their cut-edge rows routed back to
this rank (loop-back: the numbers exchanged are its own rows, the data path
and timing are the single-launch step's).  Reports ms per step and the
implied weak / strong efficiency of the per-GPU step (no NVLink latency).
usage: python tools/scaling_step_sim.py [c3|c4|c2|c5|c3x8] [--tf32]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TF32

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
fl = FLAG_GRAPH | (FLAG_TF32 if "--tf32" in sys.argv else 0)
base = None
for n in (1, 2, 4, 8):
    prob, owner, scaling = bench.workload(wl, "cpinn" if wl == "c2" else "xpinn", n)
    local = [q for q in range(prob.n_sub) if owner[q] == 0]
    cut = any(owner[prob.edge_neighbor(q, e)] != 0 for q in local for e in prob.subdomains[q].edges)
    kw = dict(transport="peer", loopback=True) if cut else {}
    h = PinnDD(prob, local, owner, 0, device="cuda:0", flags=fl, **kw)
    K = 20 if wl == "c4" else 300
    h.step(10, want_loss=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h.stream)
    h.step(K, want_loss=False)
    e1.record(h.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    base = base or ms
    eff = base / ms / n if scaling == "strong" else base / ms
    print(json.dumps(dict(workload=prob.name, n_gpus=n, local_subdomains=len(local), points=h.n_points,
                          peer_rows=int(h.table.plan.n_recv), ms_per_step=ms, step_efficiency=eff, scaling=scaling,
                          fused=h.step_fused, tf32="--tf32" in sys.argv)), flush=True)
    h.close()
