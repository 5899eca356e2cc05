import sys
import numpy as np, torch
sys.path.insert(0, ".")
from pinn_inputs import make_config
from paper_2104_10013_b200.binding import PinnDD
prob = make_config("C2", n_f=300, n_i=25, n_u=20)
m = PinnDD(prob, device="cuda:0", flags=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
p0 = m.debug_buffer(0).cpu().numpy(); c1 = m.debug_buffer(3).cpu().numpy().reshape(-1, 4); c2 = m.debug_buffer(4).cpu().numpy().reshape(-1, 4)
print("n_points", m.n_points, "chunks1", c1.shape, "chunks2", c2.shape, "plan", m.plan_info())
print("pinfo kinds", np.bincount(p0 & 3))
m.interface_payload(); torch.cuda.synchronize()
p1 = m.debug_buffer(0).cpu().numpy()
print("after K2: pinfo changed at", np.nonzero(p0 != p1)[0][:20], (p0 != p1).sum())
print("c1 changed", (m.debug_buffer(3).cpu().numpy().reshape(-1,4) != c1).sum())
try:
    loss, grad = m.loss_grad(); torch.cuda.synchronize()
    print("loss", loss[:3, :5].tolist())
except Exception as e:
    print("K1 failed", e)
