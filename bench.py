#!/usr/bin/env python
"""Benchmark of the parallel cPINN / XPINN training step (arXiv 2104.10013) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2|c3|c5] [--method cpinn|xpinn|hybrid|dp]

Default workload (BASELINE.json configs[3], "C4", the largest single-GPU
config): 2-D steady incompressible Navier-Stokes (lid-driven cavity, Re 100)
XPINN on a 4 x 2 decomposition of [0,1]^2, 5 x 80 tanh networks with outputs
(u, v, p), 125,000 residual + 80 boundary + 250 per interface edge points per
subdomain (1,005,640 points per step).  Strong scaling: the 8 subdomains are
split into contiguous blocks, 8/N per GPU.  Other workloads: c2 (configs[1],
Poisson 4x4 6x40, strong: 16/N subdomains per GPU), c3 (configs[2], Burgers
x-t XPINN 5x20, weak: one 20k-point subdomain per GPU on a 1x1 / 2x1 / 2x2 /
4x2 grid), c5 (configs[4], inverse heat on the 10-region map, LPT placement).

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


def block_owner(prob, world):
    """Contiguous Cartesian blocks of the subdomain grid, one per GPU, with the
    block grid (gx, gy), gx * gy = world, that cuts the fewest edges (SURVEY
    8(e): C2 at 8 GPUs -> 1 x 2 blocks, 16 of 24 edges cut)."""
    nx, ny = prob.nx, prob.ny
    best = None
    for gx in range(1, world + 1):
        if world % gx or nx % gx or ny % (world // gx):
            continue
        gy = world // gx
        cut = (gx - 1) * ny + (gy - 1) * nx
        if best is None or cut < best[0]:
            best = (cut, gx, gy)
    if best is None:
        raise SystemExit(f"{prob.name}: {nx} x {ny} subdomains do not split into {world} blocks")
    _, gx, gy = best
    bx, by = nx // gx, ny // gy
    return [(s.ix // bx) + gx * (s.iy // by) for s in prob.subdomains]


def workload(name, method, world):
    """(problem, owner per subdomain, scaling) of a bench workload at `world` GPUs."""
    from pinn_inputs import make_config
    if name == "c3":
        prob = make_config("C3", method=method, gpus=world)        # one subdomain per GPU
        return prob, list(range(prob.n_sub)), "weak"
    if name == "c3x8":
        # SURVEY 8(d) C3 variant: 8 subdomains (a 4 x 2 x-t block, 20k residual points
        # each) per GPU, blocks side by side in x: (4N) x 2 subdomains on [-1, 1] x [0, 1]
        prob = make_config("C3", method=method, gpus=8, nx=4 * world, ny=2)
        return prob, [s.ix // 4 for s in prob.subdomains], "weak"
    if name == "c5":
        prob = make_config("C5", method=method)
        return prob, lpt_owner([prob.n_points(q) for q in range(prob.n_sub)], world), "strong"
    prob = make_config(name.upper(), method=method)
    return prob, block_owner(prob, world), "strong"


def host_cpu():
    """Host cores this process may use and the CPU model (lscpu)."""
    cores = len(os.sched_getaffinity(0))
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


def algorithmic_bytes(prob, local, nf):
    """HBM bytes one K1 launch must move at minimum: point coordinates (8 B),
    targets + masks of data points (2 D_o x 4 B), payload rows read at
    interface points (n_fields x 4 B), and per subdomain the parameters read
    (4 B each; gradient partials are L2-resident)."""
    P = prob.sizes
    from pinn_inputs import n_params
    b = 0
    for q in local:
        s = prob.subdomains[q]
        ni = sum(len(prob.edges[e].pts) for e in s.edges)
        b += 8 * (len(s.x_f) + len(s.x_u) + ni) + 8 * prob.d_out * len(s.x_u) + 4 * nf * ni
        b += 4 * n_params(P)
    return b


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

def sample_problem(prob, q, n_res):
    """Subdomain q of `prob` with its residual points cut to the first n_res
    (uniform i.i.d. samples, so any prefix is a uniform sample); its data and
    interface points and every other subdomain unchanged."""
    import dataclasses
    s = prob.subdomains[q]
    subs = list(prob.subdomains)
    subs[q] = dataclasses.replace(s, x_f=s.x_f[:n_res])
    return dataclasses.replace(prob, subdomains=subs)


def oracle_sample_step(prob, st, q, n_res=None):
    """Loss + gradient + Adam of subdomain q (residual points cut to n_res)
    with its neighbours' payloads, FP64 oracle; returns the points processed."""
    from oracle import loss as OL
    import torch
    if n_res is not None and n_res < len(prob.subdomains[q].x_f):
        prob = sample_problem(prob, q, n_res)
    pay = {}
    for e in prob.subdomains[q].edges:
        nb = prob.edge_neighbor(q, e)
        ed = prob.edges[e]
        pay[(nb, e)] = OL.interface_payload(prob, st.thetas[nb].detach(),
                                            torch.as_tensor(ed.pts, dtype=torch.float64), ed.normal,
                                            create_graph=False, q=nb)
    bd, g = OL.loss_and_grad(prob, q, st.thetas, pay)
    th, ad = OL.adam_step(st.thetas[q], g, st.adam[q], prob.lr, prob.beta1, prob.beta2, prob.eps)
    st.thetas[q] = th
    st.adam[q] = ad
    return prob.n_points(q)


def oracle_sample_size(prob, seconds):
    """Residual points per oracle sample step so that one step takes about
    `seconds` (the FP64 oracle runs ~4-5 GFLOP/s on a 16-core host)."""
    f = flops_per_point(prob.width, prob.n_hidden, prob.d_out)
    return int(max(200, min(max(len(s.x_f) for s in prob.subdomains), seconds * 4e9 / f)))


def cpu_baseline(prob, budget_s: float = 20.0):
    """The oracle as it stands, on the host cores: full synchronous steps of
    the whole decomposition while they fit the budget, else loss + gradient +
    Adam of single subdomains (cycling) on a bounded residual-point sample."""
    import torch
    from oracle import loss as OL
    cores, model = host_cpu()
    info = {"unit": UNIT, "cores": cores, "threads": torch.get_num_threads(), "cpu_model": model,
            "kind": "oracle"}
    st = OL.init_state(prob)
    full_cost = flops_per_point(prob.width, prob.n_hidden, prob.d_out) * prob.n_points()
    if full_cost > budget_s * 4e9:
        n_res = oracle_sample_size(prob, 4.0)
        t0 = time.perf_counter()
        pts = k = 0
        while k == 0 or time.perf_counter() - t0 < budget_s:
            pts += oracle_sample_step(prob, st, k % prob.n_sub, n_res)
            k += 1
        dt = time.perf_counter() - t0
        return {"value": pts / dt, **info,
                "sample": f"{k} FP64 oracle loss+grad+Adam step(s) of single subdomains of {prob.name} "
                          f"{prob.method} (cycling), residual points cut to {n_res} per subdomain, with the "
                          f"neighbours' payloads ({pts} pts), {dt:.1f} s"}
    t0 = time.perf_counter()
    steps = 0
    while True:
        st, _ = OL.train_step(prob, st)
        steps += 1
        if time.perf_counter() - t0 >= budget_s or steps >= 10:
            break
    dt = time.perf_counter() - t0
    pts = prob.n_points() * steps
    return {"value": pts / dt, **info,
            "sample": f"{steps} full FP64 oracle step(s) of {prob.name} {prob.method} "
                      f"({prob.n_sub} subdomains, {prob.n_points()} pts/step), {dt:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from oracle import loss as OL
    prob, owner, scaling = workload(args.workload, args.method, args.gpus)
    # each step: one subdomain (cycling), residual points cut so that the whole
    # --steps K --warmup W run stays within ~2 minutes
    n_res = oracle_sample_size(prob, min(1.0, 120.0 / max(1, args.steps + args.warmup)))
    st = OL.init_state(prob)
    for w in range(args.warmup):
        oracle_sample_step(prob, st, w % prob.n_sub, n_res)
    t0 = time.perf_counter()
    pts = 0
    for k in range(args.steps):
        pts += oracle_sample_step(prob, st, k % prob.n_sub, n_res)
    dt = time.perf_counter() - t0
    val = pts / dt
    cores, model = host_cpu()
    sample = (f"per step: FP64 oracle loss+grad+Adam of ONE subdomain of {prob.name} {prob.method} (cycling), "
              f"residual points cut to {n_res}, with its neighbours' payloads; {args.steps} steps, {pts} pts, "
              f"{dt:.1f} s")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(1, args.steps), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{prob.name} {prob.method} (oracle sample)", "subdomains": prob.n_sub,
                       "net": f"2-{prob.width}x{prob.n_hidden}-{prob.d_out} tanh"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "threads": torch.get_num_threads(),
                             "cpu_model": model, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist
    import __graft_entry__ as ge
    ge.build()
    from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TIMING, FLAG_TF32

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    dp = None
    transport = None
    if args.method == "dp":
        # data-parallel vanilla PINN comparator: one 6x40 network on
        # [0,G]x[0,1] with C2's point count per GPU, points sharded, gradient all-reduce
        from paper_2104_10013_b200.binding import DataParallelPINN
        from pinn_inputs import make_config
        prob = make_config("C2", method="pinn", weak=world, nx=1, ny=1,
                           n_f=16 * 15000 * world, n_u=960 * world)
        scaling = "weak"
        dp = DataParallelPINN(prob, rank, world, device=dev, group=group, flags=0)
        dpt = DataParallelPINN(prob, rank, world, device=dev, group=group, flags=FLAG_TIMING)
        h, ht, local = dp.h, dpt.h, [0]
        h_prob = dp.h.prob
    else:
        prob, owner, scaling = workload(args.workload, args.method, world)
        local = [q for q in range(prob.n_sub) if owner[q] == rank]
        # N > 1: the library's NCCL transport, the whole iteration (exchange
        # included) one CUDA graph; N = 1: the fused single-GPU graph
        fl = FLAG_GRAPH | (FLAG_TF32 if args.tf32 else 0)
        transport = args.transport if world > 1 else None

        def make(flags, tr):
            xp = dict(transport=tr, world=world, group=group) if tr else {}
            return PinnDD(prob, local, owner, rank, device=dev, flags=flags, **xp)
        try:
            h = make(fl, transport)
        except Exception as e:
            if transport != "peer":
                raise
            # CUDA IPC between the ranks unavailable: every rank falls back to NCCL together
            print(f"[bench] peer stores unavailable ({e}); NCCL transport", file=sys.stderr)
            transport = "nccl"
            h = make(fl, transport)
        # a second handle with event-record nodes in its graph: per-kernel times
        # (K1 roofline, compute / exchange split) in their own timed region, so
        # the headline timing carries no event nodes
        ht = make(fl | FLAG_TIMING, transport)
        h_prob = prob
    stream = h.stream
    pts_local = h.n_points

    def step(hh, dpp):
        if dpp is not None:
            dpp.step(1)
        else:
            hh.step(1, want_loss=False)

    def timed_region(hh, dpp, n_steps, flush):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(n_steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(n_steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for k in range(n_steps):
            flush.zero_()                                  # L2 flush, outside the events
            starts[k].record(stream)
            step(hh, dpp)
            ends[k].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]

    for _ in range(args.warmup):
        step(h, dp)
    torch.cuda.synchronize(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.5)                                        # let nvidia-smi start sampling
    step_ms = timed_region(h, dp, args.steps, flush)
    clk = clocks.stop()
    t_ms = sum(step_ms)
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

    # ---- per-kernel breakdown: the same workload on the timing handle
    dpt_ = dpt if dp is not None else None
    for _ in range(args.warmup):
        step(ht, dpt_)
    ht.kernel_times()                                      # reset counters
    n_t = max(3, min(args.steps, 100))
    tstep_ms = timed_region(ht, dpt_, n_t, flush)
    kt = ht.kernel_times()   # K2, K1, K5, launches, exchange, K1 interior, K1 interface, exposed wait (ms)
    if dp is not None:
        kt[1] = kt[1]                                      # loss_grad calls are phased: K1 accumulated per call

    # ---- end to end through the public API with host buffers (pinned H2D + D2H loss)
    host = [h.coords.cpu().pin_memory(), h.target.cpu().pin_memory(), h.mask.cpu().pin_memory()]
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = h.n_sub * 8 * 4
    e2e_steps = max(3, min(args.steps, 50))
    # step k+1's inputs travel host -> device staging on a copy stream while step
    # k computes; each step copies staging -> the point table (device), runs,
    # and enqueues its loss read-back into pinned host memory (pinn_dd_read_loss);
    # one synchronisation at the end
    cs = torch.cuda.Stream(dev)
    staging = [torch.empty_like(t, device=dev) for t in host]
    loss_host = torch.empty(e2e_steps + 3, h.n_sub, 8, dtype=torch.float32).pin_memory()
    ev_in = [torch.cuda.Event() for _ in range(e2e_steps + 3)]
    ev_free = [torch.cuda.Event() for _ in range(e2e_steps + 3)]
    dst = [h.coords, h.target, h.mask]

    def run_e2e(k0, n):
        for k in range(k0, k0 + n):
            with torch.cuda.stream(cs):
                if k > k0:
                    cs.wait_event(ev_free[k - 1])
                for sbuf, src in zip(staging, host):
                    sbuf.copy_(src, non_blocking=True)
                ev_in[k].record(cs)
            stream.wait_event(ev_in[k])
            with torch.cuda.stream(stream):
                for d_, sbuf in zip(dst, staging):
                    d_.copy_(sbuf, non_blocking=True)
                ev_free[k].record(stream)
            step(h, dp)
            h.read_loss(loss_host[k])                      # D2H of the loss breakdown (async)

    run_e2e(0, 3)                                          # untimed warm-up of the e2e loop
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    run_e2e(3, e2e_steps)
    torch.cuda.synchronize(dev)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if not bool(torch.isfinite(loss_host[:, :, 4]).all()):
        raise SystemExit("non-finite loss in the e2e run")
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = float(pts_all.item()) * e2e_steps / float(e2e_s.item())

    # ---- roofline of the dominant kernel (K1, fused loss + grad)
    k1_flops, k2_flops = algorithmic_flops(h_prob, local)
    fused = dp is None and ht.step_fused
    if fused:
        k1_flops += k2_flops          # the fused step runs K2's payload chunks inside K1
    k1_ms = kt[1] / n_t
    k1_what = ("K1 per step, event-record nodes inside the step graph of a timing handle, over its own "
               f"timed region of {n_t} steps of the same workload")
    peak_fp32 = 148 * 128 * 2 * 1965e6 / 1e12              # TFLOP/s, FP32 FMA pipe at clocks.max.sm
    achieved = k1_flops / (k1_ms * 1e-3) / 1e12
    # HBM side of the roofline (not the bound): algorithmic bytes per K1 launch
    # and the ncu DRAM traffic, both per K1 time, vs the measured copy bandwidth
    hbm_peak, hbm_src = 6547.8, "MEASURED_PEAKS.json hbm_gbs"
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm_src = "MEASURED_PEAKS.json absent: this pool's measured 6547.8 GB/s"
    alg_bytes = algorithmic_bytes(h_prob, local, h.n_fields)
    # DRAM bytes per K1 launch of THIS workload from one committed ncu --set full
    # capture (tools/dram_table.py); null when no capture of this workload exists
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_dram_bytes.json")
    wl_key = f"{h_prob.name} {'data-parallel PINN' if dp is not None else h_prob.method}" + \
        (" tf32" if args.tf32 else "")
    if os.path.exists(prof) and world == 1:
        try:
            ent = json.load(open(prof)).get(wl_key)
            traffic = ent.get("dram_bytes_per_launch") if ent else None
        except Exception:
            traffic = None
    # compute / exchange split per step, max over ranks
    split = torch.tensor([kt[0] / n_t, kt[1] / n_t, kt[2] / n_t, kt[4] / n_t, kt[7] / n_t], dtype=torch.float64,
                         device=dev)
    if world > 1:
        dist.all_reduce(split, op=dist.ReduceOp.MAX)
    split = split.tolist()

    if rank == 0:
        base = None
        if world == 1 and not args.no_cpu and dp is None:
            base = cpu_baseline(prob)
        acts = sorted({h_prob.act(q) for q in local})
        kname = (f"K1 k_fused{'_tc' if args.tf32 else ''}<{h_prob.width},{h_prob.n_hidden},{h_prob.d_out},"
                 f"{'mixed' if len(acts) > 1 else acts[0]}> (fused fwd jets + loss + reverse"
                 f"{'; K2 interface payload in the same launch' if fused else ''})")
        share = k1_ms / (sum(tstep_ms) / n_t)
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                "frac": achieved / peak_fp32, "traffic": traffic,
                "peak_source": "148 SM x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md clocks.max.sm)"}
        if args.tf32:
            # tensor-core mode: the hidden-layer contractions (forward, input
            # adjoint, dW: 3 x (NH-1) x 2 C N^2 FLOP per point with C jets) run as
            # tcgen05 kind::tf32 MMAs; roofline against the dense TF32 peak = the
            # measured dense BF16 peak x the nominal TF32 / BF16 ratio 1/2
            try:
                bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
                src = "MEASURED_PEAKS.json bf16_tflops x 1/2 (nominal TF32 / BF16 ratio)"
            except Exception:
                bf16, src = 2250.0, "nominal 2.25 PFLOP/s BF16 x 1/2 (MEASURED_PEAKS.json absent)"
            N, NH = h_prob.width, h_prob.n_hidden
            gemm = 0.0
            for q in local:
                s_ = h_prob.subdomains[q]
                ni = sum(len(h_prob.edges[e].pts) for e in s_.edges)
                cf = 2 if h_prob.method == "cpinn" else 4
                gemm += (len(s_.x_f) * 4 + len(s_.x_u) * 1 + ni * cf) * 3 * (NH - 1) * 2 * N * N
                gemm += ni * cf * (NH - 1) * 2 * N * N if fused else 0       # K2's forward in the fused launch
            ach_t = gemm / (k1_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": ach_t, "peak": bf16 / 2, "unit": "TFLOP/s",
                    "frac": ach_t / (bf16 / 2), "traffic": traffic, "peak_source": src,
                    "tensor_gflop_per_launch": gemm / 1e9,
                    "alu_view": {"achieved_all_flops": achieved, "fp32_peak": peak_fp32,
                                 "frac": achieved / peak_fp32}}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "tf32" if args.tf32 else "f32",
            "data": "synthetic",
            "iters_per_s": 1e3 * args.steps / t_max,
            "step_ms": {"median": statistics.median(step_ms), "p10": float(np.percentile(step_ms, 10)),
                        "p90": float(np.percentile(step_ms, 90))},
            "residual_points_per_s": res_all * args.steps / (t_max * 1e-3),   # N_F only (the paper's count)
            "config": {"workload": f"{h_prob.name} {'data-parallel PINN' if dp is not None else h_prob.method}",
                       "subdomains": h_prob.n_sub,
                       "subdomains_per_gpu": len(local), "points_per_step": int(pts_all.item()),
                       "net": f"2-{h_prob.width}x{h_prob.n_hidden}-{h_prob.d_out} {'/'.join(acts)}, "
                              "adaptive slope n=10",
                       "parallelism": (f"domain decomposition, {len(local)} subdomains/GPU, neighbour-only exchange "
                                       + ("by peer stores inside the fused launch (CUDA IPC over NVLink)"
                                          if transport == "peer" else "by NCCL send/recv inside the step graph")
                                       if world > 1 and dp is None else
                                       f"domain decomposition, {len(local)} subdomains/GPU"
                                       if dp is None else "data-parallel replicas, gradient all-reduce"),
                       "l2": "flushed (256 MiB write) between timed steps"},
            "roofline": {**roof,
                         "kernel": kname,
                         "k1_ms_per_launch": k1_ms, "k1_timing": k1_what, "k1_gflop_per_launch": k1_flops / 1e9,
                         "k1_share_of_step": share,
                         "hbm": {"algorithmic_bytes_per_launch": alg_bytes,
                                 "algorithmic_gbs": alg_bytes / (k1_ms * 1e-3) / 1e9,
                                 "traffic_gbs": (traffic / (k1_ms * 1e-3) / 1e9) if traffic else None,
                                 "peak_gbs": hbm_peak, "peak_source": hbm_src,
                                 "frac": (traffic if traffic else alg_bytes) / (k1_ms * 1e-3) / 1e9 / hbm_peak,
                                 "frac_of": "ncu DRAM traffic" if traffic else "algorithmic bytes"}},
            "kernels_ms_per_step": {"K2_payload": split[0], "K2_inside_K1": fused, "K1_loss_grad": split[1],
                                    "K5_reduce_adam": split[2], "exchange": split[3],
                                    "exchange_exposed": split[4], "timing_steps": n_t,
                                    "how": "event-record nodes in the step graph of the timing handle; max over "
                                           "ranks; exchange = NCCL group on the exchange stream from the end of "
                                           "K2, exposed = wait of the compute stream after K1 interior"},
            "gpu_launches": int(kt[3] * args.steps / n_t),
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": ("pinned H2D of step k+1's point table on a copy stream overlapping step k, "
                            "device copy into the table, the step, async D2H of the loss breakdown "
                            "(pinn_dd_read_loss); one sync at the end; wall clock, max over ranks"),
                    "steps": e2e_steps},
            "cpu_baseline": base,
        }
        print(json.dumps(line))
    if dp is not None:
        dp.close()
        dpt.close()
    else:
        h.close()
        ht.close()
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
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N > 1: cut-edge rows by stores into the neighbours' memory inside the fused launch "
                         "(default), or NCCL send/recv captured in the step graph")
    ap.add_argument("--tf32", action="store_true",
                    help="hidden layers on the tensor cores (PINN_DD_FLAG_TF32, width-80 workloads c4 / c5)")
    ap.add_argument("--workload", choices=["c2", "c3", "c3x8", "c4", "c5"], default="c4",
                    help="c4: BASELINE configs[3] (default: the largest single-GPU config, strong); "
                         "c2: configs[1] (strong, 16/N subdomains per GPU); c3: configs[2] (weak, one "
                         "subdomain per GPU); c3x8: its variant with a 4x2 block of subdomains per GPU "
                         "(weak); c5: configs[4] (LPT placement, strong)")
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
