"""Multi-rank exchange (Algorithm 1 green stage) on CPU with
gloo, world_size 2: the same `exchange_payload` + `build_point_table` routing the
GPU path runs over NCCL.  Each rank fills its payload rows with a function of
the row's coordinates; after the exchange every receive row must hold the
value computed from the coordinates of the twin point the library will read."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tag(xy):
    # payload stand-in: two fields that identify the point
    return np.stack([np.sin(3.0 * xy[0]) + xy[1], xy[0] * xy[1] - 0.5], axis=1).astype(np.float32)


def _worker(rank, world, port, method, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2104_10013_b200.binding import build_point_table, exchange_payload
        from pinn_inputs import make_config
        prob = make_config("C2", method=method, weak=world, scale=0.01)
        owner = [s.ix // 4 for s in prob.subdomains]
        local = [i for i in range(prob.n_sub) if owner[i] == rank]
        t = build_point_table(prob, local, owner, rank)
        n = t.coords.shape[1]
        payload = torch.zeros(n + t.plan.n_recv, 2)
        payload[:n] = torch.from_numpy(_tag(t.coords))
        exchange_payload(payload, t.plan)
        # every interface segment's twin rows must carry the twin's (= own) coordinates' tag
        pos = 0
        bad = 0
        for qi in range(len(local)):
            pos = int(t.sub_off[qi] + t.n_res[qi] + t.n_data[qi])
            for si in range(t.seg_off[qi], t.seg_off[qi + 1]):
                m = int(t.seg_n[si])
                tw = int(t.seg_twin[si])
                want = _tag(t.coords[:, pos:pos + m])
                got = payload[tw:tw + m].numpy()
                bad += int(not np.array_equal(got, want))
                pos += m
        n_remote = int(sum(1 for tw in t.seg_twin if tw >= n))
        q.put((rank, bad, n_remote, t.plan.n_recv))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), -1, -1))


@pytest.mark.parametrize("method", ["cpinn", "xpinn"])
def test_exchange_world_size_2(method):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, method, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, bad, n_remote, n_recv in res:
        assert bad == 0, (rank, bad)
        assert n_remote == 4, (rank, n_remote)        # 4 cut edges between the two 4x4 blocks
        assert n_recv == 4 * max(1, round(250 * 0.01)), (rank, n_recv)


def _worker_strong(rank, world, port, cfg, q):
    """bench.py's strong-scaling placement (contiguous blocks of the fixed
    decomposition) through the same routing."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        from paper_2104_10013_b200.binding import build_point_table, exchange_payload
        from pinn_inputs import make_config
        prob = make_config(cfg, scale=0.01)
        owner = bench.block_owner(prob, world)
        local = [i for i in range(prob.n_sub) if owner[i] == rank]
        t = build_point_table(prob, local, owner, rank)
        n = t.coords.shape[1]
        payload = torch.zeros(n + t.plan.n_recv, 2)
        payload[:n] = torch.from_numpy(_tag(t.coords))
        exchange_payload(payload, t.plan)
        bad = 0
        for qi in range(len(local)):
            pos = int(t.sub_off[qi] + t.n_res[qi] + t.n_data[qi])
            for si in range(t.seg_off[qi], t.seg_off[qi + 1]):
                m = int(t.seg_n[si])
                tw = int(t.seg_twin[si])
                bad += int(not np.array_equal(payload[tw:tw + m].numpy(), _tag(t.coords[:, pos:pos + m])))
                pos += m
        n_remote = int(sum(1 for tw in t.seg_twin if tw >= n))
        q.put((rank, bad, n_remote, len(local)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), -1, -1))


@pytest.mark.parametrize("cfg,cut", [("C2", 4), ("C4", 2)])
def test_exchange_strong_placement_world_size_2(cfg, cut):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_strong, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, bad, n_remote, n_local in res:
        assert bad == 0, (rank, bad)
        assert n_remote == cut, (rank, n_remote)     # C2: 4x4 split in 2x4 halves; C4: 4x2 in 2x2 halves
        assert n_local * world in (16, 8)


@pytest.mark.parametrize("cfg,kw", [("C2", dict(method="xpinn")), ("C2", dict(method="cpinn")),
                                    ("C4", dict()), ("C3", dict(gpus=8))])
def test_loopback_plan_routes_every_twin(cfg, kw):
    """Loop-back plan (one process exchanging with itself, the single-GPU
    validation of the library's NCCL path): NCCL moves each peer's send rows,
    in order, into its received range; afterwards every segment's twin rows
    hold the neighbour's own rows."""
    import bench
    from paper_2104_10013_b200.binding import build_point_table
    from pinn_inputs import make_config
    prob = make_config(cfg, scale=0.01, **kw)
    owner = bench.block_owner(prob, 2)
    t = build_point_table(prob, list(range(prob.n_sub)), owner, 0, peer_of=lambda o: 0)
    n = t.coords.shape[1]
    assert set(t.plan.send) == {0} and set(t.plan.recv) == {0}
    payload = np.zeros((n + t.plan.n_recv, 2), np.float32)
    payload[:n] = _tag(t.coords)
    r0, m = t.plan.recv[0]
    assert r0 == n and m == t.plan.n_recv == len(t.plan.send[0])
    payload[r0:r0 + m] = payload[t.plan.send[0]]           # what ncclSend/ncclRecv to self does
    n_remote = 0
    for qi, q in enumerate(t.local):
        pos = int(t.sub_off[qi] + t.n_res[qi] + t.n_data[qi])
        for si in range(t.seg_off[qi], t.seg_off[qi + 1]):
            k = int(t.seg_n[si])
            tw = int(t.seg_twin[si])
            n_remote += tw >= n
            assert np.array_equal(payload[tw:tw + k], _tag(t.coords[:, pos:pos + k])), (q, si)
            pos += k
    assert n_remote > 0
