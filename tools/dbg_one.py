"""Run one loss+grad of a named small config through the ABI (debug helper)."""
import sys, json
import torch
sys.path.insert(0, ".")
from pinn_inputs import make_config
from paper_2104_10013_b200.binding import PinnDD, FLAG_GLOBAL_STASH
cfg = sys.argv[1]
kw = {k: (int(v) if v.lstrip("-").isdigit() else v) for k, v in (a.split("=") for a in sys.argv[2].split(",") if a)} if len(sys.argv) > 2 else {}
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
prob = make_config(cfg, **kw)
m = PinnDD(prob, device="cuda:0", flags=flags)
m.interface_payload(); torch.cuda.synchronize(); print("payload ok")
loss, grad = m.loss_grad(); torch.cuda.synchronize(); print("loss ok", loss[:2, :5].tolist())
