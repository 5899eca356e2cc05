"""Train a reduced C2 Poisson cPINN/XPINN on the GPU through the C ABI and report the
stitched (Eq. 4) relative L2 error against u* = sin(pi x) sin(pi y)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
from pinn_inputs import make_config
from paper_2104_10013_b200.binding import PinnDD
method = sys.argv[1] if len(sys.argv) > 1 else "cpinn"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
lr = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-3
prob = make_config("C2", method=method, n_f=2000, n_i=60, n_u=80, lr=lr)
m = PinnDD(prob, device="cuda:0")
g = np.linspace(0, 1, 101).astype(np.float32)
X = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
own = np.full((len(X), 4), -1, np.int32)
for i, (x, y) in enumerate(X):
    o = [s.id for s in prob.subdomains if s.lo[0] <= x <= s.hi[0] and s.lo[1] <= y <= s.hi[1]]
    own[i, :len(o)] = o
pts = torch.tensor(X.T.copy(), device="cuda:0"); owners = torch.tensor(own, device="cuda:0")
ref = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1])
hist = []
t0 = time.time()
for k in range(0, iters, 500):
    loss = m.step(500)
    u = m.predict(pts, owners).cpu().numpy()[0]
    err = float(np.linalg.norm(u - ref) / np.linalg.norm(ref))
    hist.append((k + 500, float(loss[:, 4].sum()), err))
    print(k + 500, "sum J", float(loss[:, 4].sum()), "rel L2", err, flush=True)
print(json.dumps({"method": method, "iters": iters, "lr": lr, "seconds": time.time() - t0, "history": hist}))
