#!/usr/bin/env python
"""Benchmark of the parallel cPINN / XPINN training step (arXiv 2104.10013) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--method cpinn|xpinn]

Workload (BASELINE.json configs[1], "C2"): 2-D Poisson on [0, G] x [0, 1], a 4 x 4
Cartesian block of subdomains per GPU (4G x 4 in total), 6 x 40 tanh networks,
per subdomain 15000 residual + 80 boundary (boundary subdomains) + 250 per
interface edge points.  G = 1 is exactly C2.  Each GPU owns one 4 x 4 block
(weak scaling); cut-edge payloads move with torch.distributed P2P (NCCL).

A "step" = one synchronous Algorithm-1 iteration over every subdomain:
interface payload (K2) -> [exchange] -> loss + gradient (K1, K5a) -> Adam (K5b).
metric = collocation-point loss+grad evaluations per second, whole job:
sum over subdomains of (N_F + N_u + sum_edges N_I) per step / step time.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on
the launching stream, L2 flushed (256 MiB write) between steps outside the
events; barrier + synchronize around the timed region; max over ranks.
The FP64 oracle (oracle/) is executed only by the cpu_baseline leg and by
--impl reference.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "collocation-pt loss+grad evals/sec (whole box) & train iters/s at 1/2/4/8 B200"
UNIT = "points/s"


# --------------------------------------------------------------------------
# algorithmic FLOPs per point, forward + reverse, C jet channels
# --------------------------------------------------------------------------

def flops_per_point(width: int, n_hidden: int, d_out: int, C: int = 4, d: int = 2,
                    reverse: bool = True) -> int:
    """fwd linear = 2 N d + (L-2) 2 C N^2 + 2 C D_o N (+ biases);
    reverse linear = 2 x (fwd linear without biases); elementwise (3d+12) fwd and
    (6d+25) rev per hidden neuron.  C = 4 reproduces the table (206,881 for 6x40)."""
    N, NH = width, n_hidden
    lin = 2 * N * d + (NH - 1) * 2 * C * N * N + 2 * C * d_out * N
    fwd = lin + NH * N + d_out + (3 * d + 12) * N * NH
    if not reverse:
        return fwd
    return fwd + 2 * lin + (6 * d + 25) * N * NH


def lpt_owner(loads, world):
    """Longest-processing-time placement: heaviest unit to the least-loaded GPU."""
    owner = [0] * len(loads)
    tot = [0] * world
    for q in sorted(range(len(loads)), key=lambda i: (-loads[i], i)):
        g = min(range(world), key=lambda r: (tot[r], r))
        owner[q] = g
        tot[g] += loads[q]
    return owner


def algorithmic_flops(prob, local):
    """K1 (loss+grad) FLOPs of one step for the local subdomains, and K2 (payload)."""
    N, NH, DO = prob.width, prob.n_hidden, prob.d_out
    f4 = flops_per_point(N, NH, DO, 4)
    f1 = flops_per_point(N, NH, DO, 1)
    fi = flops_per_point(N, NH, DO, 2 if prob.method == "cpinn" else 4)
    fwd_i = flops_per_point(N, NH, DO, 2 if prob.method == "cpinn" else 4, reverse=False)
    k1 = k2 = 0
    for q in local:
        s = prob.subdomains[q]
        ni = sum(len(prob.edges[e].pts) for e in s.edges)
        k1 += len(s.x_f) * f4 + len(s.x_u) * f1 + ni * fi
        k2 += ni * fwd_i
    return k1, k2


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.f.name)
        if sm:
            loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
            out = {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                   "samples": len(sm)}
        return out


# --------------------------------------------------------------------------
# oracle legs (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------

def oracle_sample_step(prob, st, q):
    """Loss + gradient + Adam of subdomain q with its neighbours' payloads, FP64 oracle."""
    from oracle import loss as OL
    import torch
    pay = {}
    for e in prob.subdomains[q].edges:
        nb = prob.edge_neighbor(q, e)
        ed = prob.edges[e]
        pay[(nb, e)] = OL.interface_payload(prob, st.thetas[nb].detach(),
                                            torch.as_tensor(ed.pts, dtype=torch.float64), ed.normal,
                                            create_graph=False)
    bd, g = OL.loss_and_grad(prob, q, st.thetas, pay)
    th, ad = OL.adam_step(st.thetas[q], g, st.adam[q], prob.lr, prob.beta1, prob.beta2, prob.eps)
    st.thetas[q] = th
    st.adam[q] = ad
    return prob.n_points(q)


def cpu_baseline(prob, budget_s: float = 20.0):
    """The oracle as it stands, on the host cores: full synchronous steps of the
    whole decomposition until ~budget_s of CPU work (at least one step)."""
    import torch
    from oracle import loss as OL
    st = OL.init_state(prob)
    if prob.n_points() > 300_000:
        # too large for full oracle steps within the budget (C4: 1M points): time
        # loss+grad+Adam of single subdomains (with their neighbours' payloads) instead
        t0 = time.perf_counter()
        pts = k = 0
        while k == 0 or time.perf_counter() - t0 < budget_s:
            pts += oracle_sample_step(prob, st, k % prob.n_sub)
            k += 1
        dt = time.perf_counter() - t0
        return {"value": pts / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                "sample": f"{k} single-subdomain FP64 oracle step(s) of {prob.name} {prob.method} "
                          f"({pts} pts), {dt:.1f} s"}
    t0 = time.perf_counter()
    steps = 0
    while True:
        st, _ = OL.train_step(prob, st)
        steps += 1
        if time.perf_counter() - t0 >= budget_s or steps >= 10:
            break
    dt = time.perf_counter() - t0
    pts = prob.n_points() * steps
    return {"value": pts / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
            "sample": f"{steps} full FP64 oracle step(s) of {prob.name} {prob.method} "
                      f"({prob.n_sub} subdomains, {prob.n_points()} pts/step), {dt:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from pinn_inputs import make_config
    from oracle import loss as OL
    prob = (make_config("C2", method=args.method, weak=args.gpus) if args.workload == "c2"
            else make_config(args.workload.upper(), method=args.method,
                             **({"gpus": 8} if args.workload == "c3" else {})))
    st = OL.init_state(prob)
    for w in range(args.warmup):
        oracle_sample_step(prob, st, w % prob.n_sub)
    t0 = time.perf_counter()
    pts = 0
    for k in range(args.steps):
        pts += oracle_sample_step(prob, st, k % prob.n_sub)
    dt = time.perf_counter() - t0
    val = pts / dt
    sample = (f"per step: loss+grad+Adam of ONE subdomain of {prob.name} {prob.method} (cycling), "
              f"with its neighbours' payloads; {args.steps} steps, {pts} pts, {dt:.1f} s")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak" if args.workload == "c2" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{prob.name} {prob.method} (oracle sample)", "subdomains": prob.n_sub,
                       "net": f"2-{prob.width}x{prob.n_hidden}-{prob.d_out} tanh"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist
    from pinn_inputs import make_config
    import __graft_entry__ as ge
    ge.build()
    from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TIMING

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # PINN_BENCH_SHARED_GPU=1: validation of the N > 1 code path on a one-GPU box
    # (every rank on cuda:0, gloo, payloads staged through the host); the line it
    # prints is marked and is never a bench number
    shared = os.environ.get("PINN_BENCH_SHARED_GPU") == "1" and world > 1
    gpu = 0 if shared else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    group = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    # per-kernel CUDA events (FLAG_TIMING) only at N = 1, where they are graph
    # nodes; the phased multi-GPU calls would synchronise the host per phase
    tflag = FLAG_TIMING if world == 1 else 0
    if args.method == "dp":
        # data-parallel vanilla PINN comparator: one 6x40 network on
        # [0,G]x[0,1] with C2's point count per GPU, points sharded, gradient all-reduce
        from paper_2104_10013_b200.binding import DataParallelPINN
        prob = make_config("C2", method="pinn", weak=world, nx=1, ny=1,
                           n_f=16 * 15000 * world, n_u=960 * world)
        dp = DataParallelPINN(prob, rank, world, device=dev, group=group, flags=tflag)
        h = dp.h
        h_prob, local = h.prob, [0]
    elif args.workload in ("c3", "c4", "c5"):
        # C3 Burgers x-t XPINN 4x2 (8 x 20k residual points), C4 NS cavity XPINN 4x2
        # (8 x 125k, the 1M-point strong-scaling case), C5 inverse heat (10-region map):
        # fixed decompositions, subdomains placed on GPUs by LPT on their point counts
        # (strong scaling)
        prob = make_config(args.workload.upper(), method=args.method,
                           **({"gpus": 8} if args.workload == "c3" else {}))
        owner = lpt_owner([prob.n_points(q) for q in range(prob.n_sub)], world)
        local = [q for q in range(prob.n_sub) if owner[q] == rank]
        h = PinnDD(prob, local, owner, rank, device=dev, flags=FLAG_GRAPH | tflag)
        h_prob = prob
    else:
        prob = make_config("C2", method=args.method, weak=world)
        owner = [s.ix // 4 for s in prob.subdomains]          # one 4x4 block per GPU
        local = [q for q in range(prob.n_sub) if owner[q] == rank]
        h = PinnDD(prob, local, owner, rank, device=dev, flags=FLAG_GRAPH | tflag)
        h_prob = prob
    stream = h.stream
    pts_local = h.n_points

    def step():
        if args.method == "dp":
            dp.step(1)
        elif world == 1:
            h.step(1, want_loss=False)
        else:
            h.step_distributed(1, group)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    h.kernel_times()                                       # reset counters
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(gpu)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.5)                                        # let nvidia-smi start sampling
    for k in range(args.steps):
        flush.zero_()                                      # L2 flush, outside the events
        starts[k].record(stream)
        step()
        ends[k].record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = sum(step_ms)
    kt = h.kernel_times()                                  # K2, K1, K5 ms over the timed steps, launches
    t_local = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    pts_all = torch.tensor([pts_local], dtype=torch.float64, device=dev)
    res_loc = torch.tensor([float(sum(len(h_prob.subdomains[q].x_f) for q in local))], dtype=torch.float64,
                           device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.all_reduce(pts_all, op=dist.ReduceOp.SUM)
        dist.all_reduce(res_loc, op=dist.ReduceOp.SUM)
    t_max = float(t_local.item())
    value = float(pts_all.item()) * args.steps / (t_max * 1e-3)
    res_all = float(res_loc.item())

    # ---- end to end through the public API with host buffers (pinned H2D + D2H loss)
    host = [h.coords.cpu().pin_memory(), h.target.cpu().pin_memory(), h.mask.cpu().pin_memory()]
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = h.n_sub * 8 * 4
    e2e_steps = max(3, min(args.steps, 50))
    if world > 1:
        dist.barrier()
    pipelined = world == 1 and args.method != "dp"
    if pipelined:
        # a handle without FLAG_TIMING (whose per-step event read-back would
        # synchronise the host every step); same problem, same initial state
        he = PinnDD(prob, local, owner, rank, device=dev, flags=FLAG_GRAPH)
        for _ in range(args.warmup):
            he.step(1, want_loss=False)
        # N = 1: step k+1's inputs travel host -> device staging on a copy stream
        # while step k computes; each step copies staging -> the point table
        # (device), runs, and enqueues its loss read-back into pinned host memory
        # (pinn_dd_read_loss); one synchronisation at the end
        cs = torch.cuda.Stream(dev)
        staging = [torch.empty_like(t, device=dev) for t in host]
        loss_host = torch.empty(e2e_steps, he.n_sub, 8, dtype=torch.float32).pin_memory()
        ev_in = [torch.cuda.Event() for _ in range(e2e_steps)]
        ev_free = [torch.cuda.Event() for _ in range(e2e_steps)]
        dst = [he.coords, he.target, he.mask]
    def run_e2e(n):
        for k in range(n):
            if pipelined:
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
                he.step(1, want_loss=False)
                he.read_loss(loss_host[k])                    # D2H of the loss breakdown (async)
                continue
            h.coords.copy_(host[0], non_blocking=True)
            h.target.copy_(host[1], non_blocking=True)
            h.mask.copy_(host[2], non_blocking=True)
            if args.method == "dp":
                dp.step(1, want_loss=True)
            else:
                h.step_distributed(1, group, want_loss=True)   # D2H of the loss breakdown

    run_e2e(3)                                             # untimed warm-up of the e2e loop
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    run_e2e(e2e_steps)
    torch.cuda.synchronize(dev)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if pipelined:
        if not bool(torch.isfinite(loss_host[:, :, 4]).all()):
            raise SystemExit("non-finite loss in the e2e run")
        he.close()
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = float(pts_all.item()) * e2e_steps / float(e2e_s.item())

    # ---- roofline of the dominant kernel (K1, fused loss + grad)
    k1_flops, k2_flops = algorithmic_flops(h_prob, local)
    fused = world == 1 and args.method != "dp" and h.step_fused
    if fused:
        k1_flops += k2_flops          # the fused step runs K2's payload chunks inside K1
    k1_ms = kt[1] / args.steps
    k1_what = "K1 per launch (CUDA events inside the timed region)"
    if world > 1:
        # K1 (+ K5a) timed with events on the launching stream after the timed region
        from paper_2104_10013_b200.binding import exchange_payload
        ts = []
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            if args.method != "dp":
                h.interface_payload()
                exchange_payload(h.payload, h.table.plan, group)
            e0.record(stream)
            h.loss_grad(want_grad=False)
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize(dev)
        k1_ms = sum(a.elapsed_time(b) for a, b in ts) / len(ts)
        k1_what = "K1 + K5a per call, events on the launching stream after the timed region"
    peak_fp32 = 148 * 128 * 2 * 1965e6 / 1e12              # TFLOP/s, FP32 FMA pipe at clocks.max.sm
    achieved = k1_flops / (k1_ms * 1e-3) / 1e12
    # DRAM bytes per K1 launch of THIS workload from one committed ncu --set full
    # capture (tools/dram_table.py); null when no capture of this workload exists
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_dram_bytes.json")
    wl_key = f"{prob.name} {'data-parallel PINN' if args.method == 'dp' else prob.method}"
    if os.path.exists(prof):
        try:
            ent = json.load(open(prof)).get(wl_key)
            traffic = ent.get("dram_bytes_per_launch") if ent else None
        except Exception:
            traffic = None

    if rank == 0:
        base = None
        if world == 1 and not args.no_cpu and args.method != "dp":
            base = cpu_baseline(make_config("C2", method=args.method) if args.workload == "c2" else
                                make_config(args.workload.upper(), method=args.method,
                                            **({"gpus": 8} if args.workload == "c3" else {})))
        acts = sorted({prob.act(q) for q in local})
        kname = (f"K1 k_fused<{prob.width},{prob.n_hidden},{prob.d_out},"
                 f"{'mixed' if len(acts) > 1 else acts[0]}> (fused fwd jets + loss + reverse"
                 f"{'; K2 interface payload in the same launch' if fused else ''})")
        share = kt[1] / max(1e-9, sum(kt[:3])) if world == 1 else k1_ms / (t_max / args.steps)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.workload == "c2" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            **({"shared_gpu_validation": "all ranks on cuda:0 over gloo: code-path check, not a bench number"}
               if shared else {}),
            "iters_per_s": 1e3 * args.steps / t_max,
            "step_ms": {"median": statistics.median(step_ms), "p10": float(np.percentile(step_ms, 10)),
                        "p90": float(np.percentile(step_ms, 90))},
            "residual_points_per_s": res_all * args.steps / (t_max * 1e-3),   # N_F only (the paper's count)
            "config": {"workload": f"{prob.name} {'data-parallel PINN' if args.method == 'dp' else prob.method}",
                       "subdomains": prob.n_sub,
                       "subdomains_per_gpu": len(local), "points_per_step": int(pts_all.item()),
                       "net": f"2-{prob.width}x{prob.n_hidden}-{prob.d_out} {'/'.join(acts)}, adaptive slope n=10",
                       "parallelism": f"domain decomposition, {len(local)} subdomains/GPU, P2P exchange",
                       "l2": "flushed (256 MiB write) between timed steps"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                         "frac": achieved / peak_fp32, "traffic": traffic,
                         "kernel": kname,
                         "k1_ms_per_launch": k1_ms, "k1_timing": k1_what, "k1_gflop_per_launch": k1_flops / 1e9,
                         "k1_share_of_step": share,
                         "peak_source": "148 SM x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md clocks.max.sm)"},
            "kernels_ms_per_step": {"K2_payload": (0.0 if fused else kt[0] / args.steps) if world == 1 else None,
                                    "K2_inside_K1": fused,
                                    "K1_loss_grad": k1_ms,
                                    "K5_reduce_adam": kt[2] / args.steps if world == 1 else None},
            "gpu_launches": int(kt[3]),
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": ("pinned H2D of step k+1's point table on a copy stream overlapping step k, "
                            "device copy into the table, pinn_dd_step, async D2H of the loss breakdown; "
                            "one sync at the end; wall clock" if pipelined else
                            "pinned H2D of the point table, step, synchronous D2H of the loss; wall clock"),
                    "steps": e2e_steps},
            "cpu_baseline": base,
        }
        print(json.dumps(line))
    h.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--method", choices=["cpinn", "xpinn", "hybrid", "dp"], default=None,
                    help="default cpinn for c2, xpinn for c5; dp = data-parallel vanilla PINN comparator "
                         "(Table 2)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--workload", choices=["c2", "c3", "c4", "c5"], default="c2",
                    help="c2: BASELINE configs[1] (default, the headline); c3/c4/c5: configs[2..4] "
                         "(fixed decompositions, strong scaling)")
    args = ap.parse_args()
    if args.method is None:
        args.method = "cpinn" if args.workload == "c2" else "xpinn"
    if args.workload != "c2" and args.method == "dp":
        raise SystemExit("--method dp is the C2 data-parallel comparator")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
