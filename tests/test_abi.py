"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and validates descriptors (no CUDA compute calls here)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2104_10013_b200 import binding
    return binding.load_library()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "pinn_dd.h")).read()
    names = sorted(set(re.findall(r"\b(pinn_dd_[a-z_0-9]+)\s*\(", hdr)))
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    from paper_2104_10013_b200 import binding
    assert sorted(binding.EXPORTS) == names


@pytest.mark.parametrize("args,expected", [((2, 20, 3, 1), 924), ((2, 20, 5, 1), 1766),
                                           ((2, 40, 6, 1), 8367), ((2, 80, 5, 3), 26408),
                                           ((2, 80, 3, 1), 13284)])
def test_n_params(lib, args, expected):
    assert lib.pinn_dd_n_params(*args) == expected


def _desc(prob, local=None, owner=None, rank=0, flags=0):
    from paper_2104_10013_b200 import binding
    local = list(range(prob.n_sub)) if local is None else local
    t = binding.build_point_table(prob, local, owner, rank)
    fake = dict(coords=0x1000, target=0x2000, mask=0x3000, init_params=0x4000)
    d, keep = binding.make_desc(prob, t, fake, 0, flags)
    return d, keep, t


def _ws(lib, d):
    n = C.c_size_t(0)
    st = lib.pinn_dd_workspace_size(C.byref(d), C.byref(n))
    return st, n.value, lib.pinn_dd_last_error(None).decode()


def test_workspace_size_valid(lib):
    from pinn_inputs import make_config
    d, keep, t = _desc(make_config("C2", scale=0.05))
    st, n, _ = _ws(lib, d)
    assert st == 0 and n > 0


def test_rejects_unsupported_shape(lib):
    from pinn_inputs import make_config
    d, keep, t = _desc(make_config("C1", scale=0.1, width=7))
    st, n, msg = _ws(lib, d)
    assert st == 2 and "not compiled" in msg


def test_rejects_cpinn_time_interface(lib):
    from pinn_inputs import make_config
    d, keep, t = _desc(make_config("C3", scale=0.01, method="cpinn", gpus=4))
    st, n, msg = _ws(lib, d)
    assert st == 1 and "time-axis" in msg


def test_rejects_bad_counts_and_twins(lib):
    from pinn_inputs import make_config
    p = make_config("C1", scale=0.1)
    d, keep, t = _desc(p)
    d.n_points = d.n_points + 1
    assert _ws(lib, d)[0] == 1
    d, keep, t = _desc(p)
    t.seg_twin[0] = 10 ** 6
    d2, keep2 = __import__("paper_2104_10013_b200.binding", fromlist=["x"]).make_desc(
        p, t, dict(coords=1, target=1, mask=1, init_params=1))
    assert _ws(lib, d2)[0] == 6


def test_point_table_layout_and_plan():
    """Twins reciprocate; remote twins get receive rows; the send/recv plans of
    two ranks mirror each other (the exchange of Algorithm 1 is consistent)."""
    from paper_2104_10013_b200 import binding
    from pinn_inputs import make_config
    p = make_config("C2", scale=0.02, method="xpinn")
    owner = [0 if s.iy < 2 else 1 for s in p.subdomains]
    tabs = [binding.build_point_table(p, [q for q in range(16) if owner[q] == r], owner, r) for r in (0, 1)]
    for r, t in enumerate(tabs):
        other = 1 - r
        n_pts = t.coords.shape[1]
        # rows sent to the peer == rows the peer receives from us (same count, edge order)
        assert len(t.plan.send[other]) == tabs[other].plan.recv[r][1]
        assert t.plan.n_recv == t.plan.recv[other][1]
        for i, tw in enumerate(t.seg_twin):
            if tw < n_pts:   # local twin points at the same coordinates
                n = t.seg_n[i]
                s0 = int(t.seg_off[0])
                # find segment start
                start = None
        # coordinates of sent rows equal those the peer expects at its receive rows
        send_xy = t.coords[:, t.plan.send[other]]
        o = tabs[other]
        r0, n = o.plan.recv[r]
        # the peer's segments whose twins are in [r0, r0+n) must have the same coordinates
        got = np.zeros((2, n), np.float32)
        seg_start = []
        pos = 0
        for qi, q in enumerate(o.local):
            pos = int(o.sub_off[qi]) + int(o.n_res[qi]) + int(o.n_data[qi])
            for si in range(o.seg_off[qi], o.seg_off[qi + 1]):
                tw = o.seg_twin[si]
                if tw >= o.coords.shape[1]:
                    got[:, tw - r0: tw - r0 + o.seg_n[si]] = o.coords[:, pos:pos + o.seg_n[si]]
                pos += o.seg_n[si]
        np.testing.assert_array_equal(send_xy, got)


def test_exchange_plan_validated(lib):
    """A loop-back / multi-rank exchange plan passes workspace_size; malformed
    plans are protocol errors (EPROTOCOL) with a message."""
    import bench
    from paper_2104_10013_b200 import binding
    from pinn_inputs import make_config
    prob = make_config("C2", method="xpinn", scale=0.02)
    owner = bench.block_owner(prob, 2)
    t = binding.build_point_table(prob, list(range(prob.n_sub)), owner, 0, peer_of=lambda o: 0)
    fake = dict(coords=0x1000, target=0x2000, mask=0x3000, init_params=0x4000)
    d, keep = binding.make_desc(prob, t, fake, 0, 0)
    assert d.n_peers == 1 and d.n_recv > 0
    st, n, msg = _ws(lib, d)
    assert st == 0, msg
    d.peer_recv_row[0] = d.peer_recv_row[0] + 1
    st, n, msg = _ws(lib, d)
    assert st == binding.EPROTOCOL and "received rows" in msg
    d.peer_recv_row[0] = d.peer_recv_row[0] - 1
    d.send_rows[0] = 10 ** 9
    st, n, msg = _ws(lib, d)
    assert st == binding.EPROTOCOL and "send row" in msg


def test_geometry_validated(lib):
    from paper_2104_10013_b200 import binding
    from pinn_inputs import make_config
    d, keep, t = _desc(make_config("C2", scale=0.02))
    assert d.geometry == binding.GEOM_BOXES and d.n_geo == 16
    st, n, msg = _ws(lib, d)
    assert st == 0, msg
    d.geo_local[3] = 99
    st, n, msg = _ws(lib, d)
    assert st == binding.EINVAL and "geo_local" in msg
