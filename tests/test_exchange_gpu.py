"""The library's NCCL transport (Algorithm 1 green stage)
and Eq. (4) classification on one GPU.

Only one GPU is available to this build, and NCCL refuses two ranks on one
device, so the multi-GPU data path is validated by LOOP-BACK: one process owns
every subdomain, but edges between two placement blocks are routed through
receive rows filled by ncclSend / ncclRecv to itself -- the same K2 send-buffer
epilogue, NCCL group, exchange stream, interior/interface split and CUDA graph
that pinn_dd_step runs with remote ranks.  It must equal the all-local fused
step bit for bit."""

import numpy as np
import pytest
import torch

from oracle import loss as OL
from oracle import net as onet
from pinn_inputs import make_config, perturb_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


def _pair(prob, blocks=2, flags=None):
    import bench
    from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH
    fl = FLAG_GRAPH if flags is None else flags
    one = PinnDD(prob, device="cuda:0", flags=fl)
    owner = bench.block_owner(prob, blocks)
    lb = PinnDD(prob, list(range(prob.n_sub)), owner, 0, device="cuda:0", flags=fl, transport="nccl",
                loopback=True)
    assert lb.table.plan.n_recv > 0 and not lb.step_fused and one.step_fused
    return one, lb


def _state(m):
    return [torch.cat([m.get(q, w) for w in (0, 1, 2, 3)]).cpu() for q in range(m.n_sub)]


@pytest.mark.parametrize("cfg,kw,blocks", [("C2", dict(method="xpinn", n_f=500, n_i=25, n_u=20), 2),
                                           ("C2", dict(method="cpinn", n_f=500, n_i=25, n_u=20), 8),
                                           ("C4", dict(method="xpinn", n_f=300, n_i=20, n_u=16), 4),
                                           ("C3", dict(method="hybrid", gpus=8, n_f=500, n_i=30, n_u=40), 8)])
def test_nccl_loopback_step_equals_local_step(cfg, kw, blocks):
    """pinn_dd_step through the NCCL path (graph-captured, 5 iterations) ==
    the all-local fused step: losses, gradients, parameters, Adam moments."""
    prob = perturb_params(make_config(cfg, **kw), scale=0.1)
    one, lb = _pair(prob, blocks)
    a = one.step(5)
    b = lb.step(5)
    torch.cuda.synchronize()
    assert np.array_equal(a, b)
    for x, y in zip(_state(one), _state(lb)):
        assert torch.equal(x, y)
    one.close()
    lb.close()


def test_nccl_loopback_phased_calls_and_timing():
    """The phased calls with the library's exchange (pinn_dd_exchange) equal
    pinn_dd_loss_grad of the all-local handle; with FLAG_TIMING the step
    reports exchange, interior and interface times."""
    from paper_2104_10013_b200.binding import FLAG_GRAPH, FLAG_TIMING
    prob = perturb_params(make_config("C2", method="cpinn", n_f=400, n_i=25, n_u=20), scale=0.1)
    one, lb = _pair(prob, 4, flags=FLAG_GRAPH | FLAG_TIMING)
    one.interface_payload()
    l1, g1 = one.loss_grad()
    lb.interface_payload()
    lb.exchange()
    l2, g2 = lb.loss_grad()
    torch.cuda.synchronize()
    assert torch.equal(l1, l2) and torch.equal(g1, g2)
    lb.kernel_times()
    lb.step(10, want_loss=False)
    kt = lb.kernel_times()
    k2, k1, k5, launches, xch, k1i, k1f, wait = kt
    assert k2 > 0 and k1 > 0 and k5 > 0 and xch > 0 and k1i > 0 and k1f > 0 and wait >= 0
    assert abs(k1 - (k1i + k1f)) < 1e-6 * max(1.0, k1)
    assert launches == 10 * 5
    one.close()
    lb.close()


def test_step_without_transport_rejects_remote_twins():
    from paper_2104_10013_b200.binding import PinnDD, PinnDDError, EPROTOCOL
    prob = make_config("C2", method="xpinn", n_f=100, n_i=10, n_u=10)
    owner = [0 if s.iy < 2 else 1 for s in prob.subdomains]
    h = PinnDD(prob, [q for q in range(16) if owner[q] == 0], owner, 0, device="cuda:0")
    with pytest.raises(PinnDDError) as ei:
        h.step(1)
    assert ei.value.status == EPROTOCOL and "NCCL" in str(ei.value)
    h.close()


# --------------------------------------------------------------------------
# Eq. (4) with the library's own classification
# --------------------------------------------------------------------------

def _cartesian_points(prob, n, seed):
    rng = np.random.default_rng(seed)
    lo, hi = np.array(prob.domain_lo), np.array(prob.domain_hi)
    X = rng.uniform(lo, hi, size=(n, 2))
    # interface, corner and outside points
    xs = [s.hi[0] for s in prob.subdomains if s.hi[0] < hi[0]]
    ys = [s.hi[1] for s in prob.subdomains if s.hi[1] < hi[1]]
    # off-corner points of every interface (0.37 of the way along the other axis is on no
    # interface of these grids), one corner, one point outside, the domain corner
    extra = [[x, lo[1] + 0.37 * (hi[1] - lo[1])] for x in xs] + [[lo[0] + 0.37 * (hi[0] - lo[0]), y] for y in ys]
    extra += [[x, y] for x in xs[:1] for y in ys[:1]] + [[lo[0] - 0.1, lo[1]], [hi[0], hi[1]]]
    return np.concatenate([X, np.array(extra)]).astype(np.float32)


@pytest.mark.parametrize("cfg,kw", [("C3", dict(method="xpinn", gpus=4, n_f=100, n_i=10, n_u=10)),
                                    ("C2", dict(method="cpinn", n_f=100, n_i=10, n_u=10)),
                                    ("C4", dict(method="xpinn", n_f=100, n_i=10, n_u=10))])
def test_predict_library_classification_cartesian(cfg, kw):
    """pinn_dd_predict classifies owners itself (closed cells; 1/S on
    interfaces, 1/4 at a 4-way corner, 0 outside) = oracle.loss.stitch."""
    prob = perturb_params(make_config(cfg, **kw), scale=0.1)
    from paper_2104_10013_b200.binding import PinnDD
    m = PinnDD(prob, device="cuda:0")
    X = _cartesian_points(prob, 300, 4)
    out = m.predict(torch.tensor(X.T.copy(), device="cuda:0")).cpu().numpy().T
    th = OL.init_state(prob).thetas
    ref = OL.stitch(prob, th, X.astype(np.float64)).numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
    own = OL.owners(prob, X.astype(np.float64))
    assert any(len(o) == 2 for o in own) and any(len(o) == 0 for o in own)
    # owner mode: the lowest-id owner's net alone
    out1 = m.predict(torch.tensor(X.T.copy(), device="cuda:0"), mode="owner").cpu().numpy().T
    Xt = torch.tensor(X.astype(np.float64))
    for i, o in enumerate(own):
        want = np.zeros(prob.d_out) if not o else \
            onet.forward(th[min(o)], prob.sizes, Xt[i:i + 1], prob.act(min(o)), prob.slope_n).numpy()[0]
        np.testing.assert_allclose(out1[i], want, rtol=1e-5, atol=1e-5)
    m.close()


def test_predict_library_classification_split_over_ranks():
    """With the subdomains split over two handles each returns its local
    owners' share (S counts every owner): the sum is the stitched field."""
    import bench
    from paper_2104_10013_b200.binding import PinnDD
    prob = perturb_params(make_config("C2", method="xpinn", n_f=100, n_i=10, n_u=10), scale=0.1)
    owner = bench.block_owner(prob, 2)
    hs = [PinnDD(prob, [q for q in range(16) if owner[q] == r], owner, r, device="cuda:0") for r in (0, 1)]
    X = _cartesian_points(prob, 200, 5)
    pts = torch.tensor(X.T.copy(), device="cuda:0")
    tot = sum(h.predict(pts) for h in hs).cpu().numpy().T
    ref = OL.stitch(prob, OL.init_state(prob).thetas, X.astype(np.float64)).numpy()
    np.testing.assert_allclose(tot, ref, rtol=1e-5, atol=1e-5)
    for h in hs:
        h.close()


def test_predict_library_classification_voronoi():
    """C5 map: owners = nearest seed(s) inside the polygon (distance tie within
    1e-5 -> 1/S), 0 outside; the test classifies independently in FP64."""
    from paper_2104_10013_b200.binding import PinnDD
    from pinn_inputs import voronoi as vor
    prob = make_config("C5", scale=0.02, n_i=10, n_u=20)
    m = PinnDD(prob, device="cuda:0")
    rng = np.random.default_rng(7)
    X = rng.uniform(prob.domain_lo, prob.domain_hi, size=(500, 2))
    X = np.concatenate([X, prob.edges[0].pts[:3], prob.edges[-1].pts[:2]]).astype(np.float32)
    out = m.predict(torch.tensor(X.T.copy(), device="cuda:0")).cpu().numpy().T
    seeds = prob.meta["seeds"]
    Xd = X.astype(np.float64)
    d = np.linalg.norm(Xd[:, None, :] - seeds[None], axis=2)
    ins = vor.inside(prob.meta["polygon"], Xd)
    own = [[] if not ins[i] else list(np.flatnonzero(d[i] <= d[i].min() + 1e-5)) for i in range(len(X))]
    assert sum(len(o) == 2 for o in own) >= 5 and sum(len(o) == 0 for o in own) >= 5
    th = OL.init_state(prob).thetas
    ref = np.zeros((len(X), 2))
    Xt = torch.tensor(Xd)
    for q in range(prob.n_sub):
        w = np.array([1.0 / len(o) if q in o else 0.0 for o in own])
        if w.any():
            ref += w[:, None] * onet.forward(th[q], prob.sizes, Xt, prob.act(q), prob.slope_n).numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)
    m.close()


# --------------------------------------------------------------------------
# peer-store transport: the exchange inside the fused persistent launch
# --------------------------------------------------------------------------

@pytest.mark.parametrize("cfg,kw,blocks,flags", [
    ("C2", dict(method="xpinn", n_f=500, n_i=25, n_u=20), 2, 0),
    ("C2", dict(method="cpinn", n_f=500, n_i=25, n_u=20), 8, 0),
    ("C3", dict(method="hybrid", gpus=8, n_f=500, n_i=30, n_u=40), 8, 0),
    ("C4", dict(method="xpinn", n_f=300, n_i=20, n_u=16), 4, 0),
    ("C4", dict(method="xpinn", n_f=300, n_i=20, n_u=16), 4, 8),          # FLAG_TF32 kernel
    ("C5", dict(scale=0.05, n_i=24, n_u=40), 2, 0),
])
def test_peer_store_loopback_step_equals_local_step(cfg, kw, blocks, flags):
    """pinn_dd_step with PINN_DD_FLAG_PEER_STORES: ONE persistent launch per
    iteration whose payload chunks store the cut-edge rows into the (here:
    own) receive slot of the step's parity and release the row counts; the
    interface loss chunks acquire-wait for them.  Seven iterations (both slot
    parities, graph-replayed) equal the all-local fused step bitwise; the
    peer launch count per iteration is the single-GPU one."""
    import bench
    from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TIMING
    prob = perturb_params(make_config(cfg, **kw), scale=0.1)
    owner = bench.block_owner(prob, blocks) if cfg != "C5" else [q % blocks for q in range(prob.n_sub)]
    one = PinnDD(prob, device="cuda:0", flags=FLAG_GRAPH | flags)
    lb = PinnDD(prob, list(range(prob.n_sub)), owner, 0, device="cuda:0", flags=FLAG_GRAPH | FLAG_TIMING | flags,
                transport="peer", loopback=True)
    assert lb.table.plan.n_recv > 0 and lb.step_fused
    a = one.step(7)
    b = lb.step(7)
    torch.cuda.synchronize()
    assert np.array_equal(a, b)
    for x, y in zip(_state(one), _state(lb)):
        assert torch.equal(x, y)
    kt = lb.kernel_times()
    assert kt[3] == 7 * 3 and kt[4] == 0.0          # fused launch + K5a + K5b, no separate exchange
    one.close()
    lb.close()
