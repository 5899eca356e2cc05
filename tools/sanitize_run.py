"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
C1 fused step, small C2 XPINN fused step (MODE 2 spin-wait), phased calls,
the TF32 tensor-core kernel on small C4, loop-back NCCL step, predict."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TF32
from pinn_inputs import make_config
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "c1"):
    m = PinnDD(make_config("C1", n_f=200, n_i=20, n_u=40), device="cuda:0", flags=0)
    m.step(2); m.interface_payload(); m.loss_grad(); m.adam(); m.close()
if which in ("all", "c2"):
    p = make_config("C2", method="xpinn", n_f=300, n_i=20, n_u=20)
    m = PinnDD(p, device="cuda:0", flags=0)
    assert m.step_fused
    m.step(2)
    pts = torch.rand(2, 100, device="cuda:0")
    m.predict(pts)
    m.close()
if which in ("all", "tf32"):
    m = PinnDD(make_config("C4", method="xpinn", n_f=300, n_i=20, n_u=16), device="cuda:0", flags=FLAG_TF32)
    m.step(2); m.interface_payload(); m.loss_grad(); m.close()
if which in ("all", "nccl"):
    import bench
    p = make_config("C2", method="cpinn", n_f=200, n_i=20, n_u=20)
    m = PinnDD(p, list(range(16)), bench.block_owner(p, 2), 0, device="cuda:0", flags=0, transport="nccl", loopback=True)
    m.step(2); m.close()
torch.cuda.synchronize()
print("sanitize workload ok", which)
if which == "c4":
    m = PinnDD(make_config("C4", method="xpinn", n_f=300, n_i=20, n_u=16), device="cuda:0", flags=0)
    m.step(2); m.close()
    torch.cuda.synchronize()
    print("c4 ok")
