"""Two ranks of the distributed Algorithm-1 step on ONE B200 (both processes
on cuda:0, gloo process group, payload rows staged through the host): K2 ->
exchange of the cut-edge payloads -> K1 interior (overlapping the exchange) ->
K1 interface + K5a -> Adam, for 3 iterations.  Every rank's parameters must be
bitwise those of the single-handle fused step on the same decomposition
(placement invariance).  NCCL itself refuses two ranks on one
GPU, so this exercises everything of the multi-GPU path except the NCCL
transport."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


ITERS = 3


def _problem():
    from pinn_inputs import make_config
    return make_config("C2", method="xpinn", weak=2, n_f=300, n_i=20, n_u=16)


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2104_10013_b200.binding import PinnDD
        prob = _problem()
        owner = [s.ix // 4 for s in prob.subdomains]
        local = [i for i in range(prob.n_sub) if owner[i] == rank]
        h = PinnDD(prob, local, owner, rank, device="cuda:0")
        loss = h.step_distributed(ITERS, dist.group.WORLD, want_loss=True)
        params = {q_: h.get(i, 0).cpu().numpy() for i, q_ in enumerate(h.table.local)}
        q.put((rank, params, loss, int(h.table.plan.n_recv)))
        h.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), None, -1))


def test_two_rank_distributed_step_matches_single_handle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    from paper_2104_10013_b200.binding import PinnDD
    prob = _problem()
    one = PinnDD(prob, device="cuda:0")
    one_loss = one.step(ITERS)
    ref = {q: one.get(q, 0).cpu().numpy() for q in range(prob.n_sub)}
    one.close()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    seen = set()
    for rank, params, loss, n_recv in sorted(res, key=lambda r: r[0]):
        assert isinstance(params, dict), params
        assert n_recv > 0, (rank, n_recv)                 # the cut edges really go through the exchange
        for q, th in params.items():
            assert np.array_equal(th, ref[q]), (rank, q, float(np.max(np.abs(th - ref[q]))))
            seen.add(q)
        loc = sorted(params)
        for i, q in enumerate(loc):
            assert np.array_equal(loss[i, :5], one_loss[q, :5]), (rank, q)
    assert seen == set(range(prob.n_sub))


def _worker_peer(rank, world, port, q):
    """Two processes on cuda:0 with the PEER-STORE transport: CUDA IPC handles
    of the exchange regions traded over gloo; each rank's fused launch stores
    its cut-edge rows into the OTHER process's receive slot and release-adds
    the counts; the interface chunks acquire-wait for them (the two processes'
    launches are time-sliced on one GPU; on a multi-GPU box they run at the
    same time on different GPUs)."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2104_10013_b200.binding import PinnDD
        prob = _problem()
        owner = [s.ix // 4 for s in prob.subdomains]
        local = [i for i in range(prob.n_sub) if owner[i] == rank]
        h = PinnDD(prob, local, owner, rank, device="cuda:0", transport="peer", world=world, group=dist.group.WORLD)
        assert h.step_fused
        loss = None
        for _ in range(ITERS):
            loss = h.step(1)
            dist.barrier()
        params = {q_: h.get(i, 0).cpu().numpy() for i, q_ in enumerate(h.table.local)}
        q.put((rank, params, loss, int(h.table.plan.n_recv)))
        dist.barrier()
        h.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), None, -1))


def test_two_process_peer_store_step_matches_single_handle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    from paper_2104_10013_b200.binding import PinnDD
    prob = _problem()
    one = PinnDD(prob, device="cuda:0")
    one_loss = one.step(ITERS)
    ref = {q: one.get(q, 0).cpu().numpy() for q in range(prob.n_sub)}
    one.close()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    procs = [ctx.Process(target=_worker_peer, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    seen = set()
    for rank, params, loss, n_recv in sorted(res, key=lambda r: r[0]):
        assert isinstance(params, dict), params
        assert n_recv > 0, (rank, n_recv)
        for q, th in params.items():
            assert np.array_equal(th, ref[q]), (rank, q, float(np.max(np.abs(th - ref[q]))))
            seen.add(q)
        for i, q in enumerate(sorted(params)):
            assert np.array_equal(loss[i, :5], one_loss[q, :5]), (rank, q)
    assert seen == set(range(prob.n_sub))
