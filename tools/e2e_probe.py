"""Development probe: end-to-end step loop variants through the public API (C2)."""
import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH
from pinn_inputs import make_config

dev = torch.device("cuda", 0)
prob = make_config("C2", method="cpinn")
for variant in ("seq", "pipe_default", "pipe_own_stream", "compute_only"):
    ctx = torch.cuda.stream(torch.cuda.Stream(dev)) if variant == "pipe_own_stream" else torch.cuda.stream(torch.cuda.current_stream(dev))
    with ctx:
        h = PinnDD(prob, device=dev, flags=FLAG_GRAPH)
        stream = h.stream
        host = [h.coords.cpu().pin_memory(), h.target.cpu().pin_memory(), h.mask.cpu().pin_memory()]
        n = 20
        cs = torch.cuda.Stream(dev)
        staging = [torch.empty_like(t, device=dev) for t in host]
        loss_host = torch.empty(n, h.n_sub, 8).pin_memory()
        ev_in = [torch.cuda.Event() for _ in range(n)]
        ev_free = [torch.cuda.Event() for _ in range(n)]
        dst = [h.coords, h.target, h.mask]
        for _ in range(5):
            h.step(1, want_loss=False)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for k in range(n):
            if variant == "compute_only":
                h.step(1, want_loss=False)
            elif variant == "seq":
                for d_, src in zip(dst, host):
                    d_.copy_(src, non_blocking=True)
                h.step(1, want_loss=True)
            else:
                with torch.cuda.stream(cs):
                    if k > 0:
                        cs.wait_event(ev_free[k - 1])
                    for sbuf, src in zip(staging, host):
                        sbuf.copy_(src, non_blocking=True)
                    ev_in[k].record(cs)
                stream.wait_event(ev_in[k])
                with torch.cuda.stream(stream):
                    for d_, sbuf in zip(dst, staging):
                        d_.copy_(sbuf, non_blocking=True)
                    ev_free[k].record(stream)
                h.step(1, want_loss=False)
                h.read_loss(loss_host[k])
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / n
        print(variant, f"{dt*1e3:.3f} ms/step", f"{h.n_points/dt:.4g} pts/s", flush=True)
        h.close()
