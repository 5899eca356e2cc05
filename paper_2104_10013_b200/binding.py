"""Thin ctypes binding of libpinn_dd.so (include/pinn_dd.h).

Argument marshalling only: every step of the training step runs in the CUDA
kernels behind the C ABI.  PyTorch supplies device memory (tensors), the CUDA
stream and, for multi-GPU runs, the process group used to move interface
payload rows between ranks (Algorithm 1 green stage).
There is NO CPU fallback: constructing `PinnDD` without a CUDA device or
without the compiled library raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PINN_DD_LIB", os.path.join(_HERE, "libpinn_dd.so"))

OK, EINVAL, EUNSUPPORTED, ECUDA, ENCCL, ENONFINITE, EPROTOCOL = range(7)
METHODS = {"pinn": 0, "cpinn": 1, "xpinn": 2, "hybrid": 3}
PDES = {"burgers": 0, "poisson": 1, "heat": 2, "ns": 3, "heat_inv": 4}
ACTS = {"tanh": 0, "sin": 1, "cos": 2}
FLAG_GRAPH, FLAG_GLOBAL_STASH, FLAG_TIMING, FLAG_TF32, FLAG_PEER_STORES = 1, 2, 4, 8, 16
GEOM_NONE, GEOM_BOXES, GEOM_VORONOI = 0, 1, 2
PREDICT_STITCHED, PREDICT_OWNER = 0, 1
STATUS_J, STATUS_GRAD, STATUS_SLOPE, STATUS_SLOPE_ZERO = 1, 2, 4, 8

EXPORTS = [
    "pinn_dd_n_params", "pinn_dd_workspace_size", "pinn_dd_create", "pinn_dd_interface_payload",
    "pinn_dd_payload_buffer", "pinn_dd_loss_grad", "pinn_dd_loss_grad_interior", "pinn_dd_loss_grad_interface",
    "pinn_dd_adam", "pinn_dd_step", "pinn_dd_predict", "pinn_dd_predict_owners", "pinn_dd_exchange",
    "pinn_dd_nccl_unique_id", "pinn_dd_ipc_export", "pinn_dd_connect_peers",
    "pinn_dd_get_params", "pinn_dd_set_params", "pinn_dd_get_step", "pinn_dd_kernel_times",
    "pinn_dd_plan_info", "pinn_dd_step_fused", "pinn_dd_read_loss", "pinn_dd_debug_buffer", "pinn_dd_destroy", "pinn_dd_last_error",
]


class PinnDDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pinn_dd status {status}: {msg}")
        self.status = status


class HParams(C.Structure):
    _fields_ = [("w_u", C.c_float), ("w_f", C.c_float), ("w_i", C.c_float), ("w_if", C.c_float),
                ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


class Desc(C.Structure):
    _fields_ = [
        ("method", C.c_int32), ("pde", C.c_int32), ("activation", C.c_int32), ("d_in", C.c_int32),
        ("d_out", C.c_int32), ("width", C.c_int32), ("n_hidden", C.c_int32),
        ("slope_n", C.c_float), ("nu", C.c_float), ("re", C.c_float),
        ("n_sub", C.c_int32),
        ("sub_point_offset", C.POINTER(C.c_int32)), ("sub_n_res", C.POINTER(C.c_int32)),
        ("sub_n_data", C.POINTER(C.c_int32)), ("sub_seg_offset", C.POINTER(C.c_int32)),
        ("sub_hparams", C.POINTER(HParams)),
        ("n_seg", C.c_int32),
        ("seg_n", C.POINTER(C.c_int32)), ("seg_normal", C.POINTER(C.c_float)),
        ("seg_twin", C.POINTER(C.c_int64)),
        ("n_points", C.c_int64), ("n_recv", C.c_int64),
        ("coords", C.c_void_p), ("target", C.c_void_p), ("mask", C.c_void_p), ("init_params", C.c_void_p),
        ("stream", C.c_void_p), ("flags", C.c_int32),
        ("sub_norm_counts", C.POINTER(C.c_int32)),
        ("sub_activation", C.POINTER(C.c_int32)),
        ("rank", C.c_int32), ("world", C.c_int32), ("n_peers", C.c_int32),
        ("peer_rank", C.POINTER(C.c_int32)), ("peer_send_off", C.POINTER(C.c_int64)),
        ("send_rows", C.POINTER(C.c_int64)), ("peer_recv_row", C.POINTER(C.c_int64)),
        ("peer_recv_n", C.POINTER(C.c_int64)), ("nccl_id", C.c_void_p),
        ("geometry", C.c_int32), ("n_geo", C.c_int32), ("geo", C.POINTER(C.c_float)),
        ("geo_local", C.POINTER(C.c_int32)), ("n_poly", C.c_int32), ("poly", C.POINTER(C.c_float)),
        ("geo_tol", C.c_float),
    ]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpinn_dd.so; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    vp, i32, i64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_float)
    lib.pinn_dd_n_params.restype = i64
    lib.pinn_dd_n_params.argtypes = [i32, i32, i32, i32]
    lib.pinn_dd_workspace_size.argtypes = [C.POINTER(Desc), C.POINTER(C.c_size_t)]
    lib.pinn_dd_create.argtypes = [C.POINTER(Desc), vp, C.c_size_t, C.POINTER(vp)]
    lib.pinn_dd_interface_payload.argtypes = [vp]
    lib.pinn_dd_payload_buffer.argtypes = [vp, C.POINTER(vp), C.POINTER(i32), C.POINTER(i64)]
    lib.pinn_dd_loss_grad.argtypes = [vp, vp, vp]
    lib.pinn_dd_loss_grad_interior.argtypes = [vp]
    lib.pinn_dd_loss_grad_interface.argtypes = [vp, vp, vp]
    lib.pinn_dd_adam.argtypes = [vp]
    lib.pinn_dd_step.argtypes = [vp, i32, f32p]
    lib.pinn_dd_predict.argtypes = [vp, vp, i64, vp, i32]
    lib.pinn_dd_predict_owners.argtypes = [vp, vp, vp, i64, vp]
    lib.pinn_dd_exchange.argtypes = [vp]
    lib.pinn_dd_nccl_unique_id.argtypes = [vp]
    lib.pinn_dd_ipc_export.argtypes = [vp, vp, C.POINTER(i64), C.POINTER(i64)]
    lib.pinn_dd_connect_peers.argtypes = [vp, vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                          C.POINTER(i32)]
    lib.pinn_dd_get_params.argtypes = [vp, i32, i32, vp]
    lib.pinn_dd_set_params.argtypes = [vp, i32, i32, vp]
    lib.pinn_dd_get_step.argtypes = [vp, i32, C.POINTER(i32)]
    lib.pinn_dd_kernel_times.argtypes = [vp, C.POINTER(C.c_double)]
    lib.pinn_dd_plan_info.argtypes = [vp, C.POINTER(i64)]
    lib.pinn_dd_read_loss.argtypes = [vp, vp]
    lib.pinn_dd_step_fused.argtypes = [vp]
    lib.pinn_dd_step_fused.restype = i32
    lib.pinn_dd_debug_buffer.argtypes = [vp, i32, C.POINTER(vp), C.POINTER(i64)]
    lib.pinn_dd_destroy.argtypes = [vp]
    lib.pinn_dd_destroy.restype = None
    lib.pinn_dd_last_error.argtypes = [vp]
    lib.pinn_dd_last_error.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("pinn_dd_n_params", "pinn_dd_destroy", "pinn_dd_last_error", "pinn_dd_step_fused"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _arr(np_arr, ctype):
    a = np.ascontiguousarray(np_arr)
    return a, a.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------------------
# host-side layout of the point table (ordering and twins only; no arithmetic)
# ---------------------------------------------------------------------------

@dataclass
class ExchangePlan:
    """Which payload rows go to / come from which rank (cut edges only)."""
    send: Dict[int, np.ndarray]            # peer -> local payload row indices (edge order)
    recv: Dict[int, Tuple[int, int]]       # peer -> (first row, n rows) in the payload buffer
    n_recv: int


@dataclass
class PointTable:
    local: List[int]                       # global subdomain ids owned here, in order
    coords: np.ndarray                     # [2, n]
    target: np.ndarray                     # [d_out, n]
    mask: np.ndarray                       # [d_out, n]
    sub_off: np.ndarray
    n_res: np.ndarray
    n_data: np.ndarray
    seg_off: np.ndarray
    seg_n: np.ndarray
    seg_normal: np.ndarray                 # [n_seg, 2]
    seg_twin: np.ndarray
    seg_edge: np.ndarray                   # global edge id of each segment
    params: np.ndarray                     # [n_local, n_params] float32
    plan: ExchangePlan


def build_point_table(prob, local: Sequence[int], owner: Optional[Sequence[int]] = None,
                      rank: int = 0, peer_of=None) -> PointTable:
    """Lay out the point sets of the `local` subdomains (global ids) in the
    order the ABI expects.  An edge is cut when its two subdomains have
    different owners; the twin of a cut edge's segment is a receive row after
    the local points, filled by the exchange with rank peer_of(owner[nb])
    (identity by default; a loop-back plan maps every owner to this rank, so a
    single process exchanges with itself).  Per peer, rows are sent in (edge,
    sender) order and received in (edge, neighbour) order, so both sides of
    every cut edge agree on the order."""
    local = list(local)
    owner = list(owner) if owner is not None else [rank] * prob.n_sub
    peer_of = peer_of or (lambda o: o)
    d_out = prob.d_out
    xs, ts, ms = [], [], []
    sub_off, n_res, n_data, seg_off = [0], [], [], [0]
    seg_n, seg_normal, seg_edge, seg_start, seg_sub = [], [], [], [], []
    pos = 0
    for q in local:
        s = prob.subdomains[q]
        parts = [s.x_f, s.x_u]
        xs.append(s.x_f); ts.append(np.zeros((len(s.x_f), d_out))); ms.append(np.zeros((len(s.x_f), d_out)))
        xs.append(s.x_u); ts.append(s.u_target); ms.append(s.u_mask)
        pos += len(s.x_f) + len(s.x_u)
        for e in s.edges:
            ed = prob.edges[e]
            xs.append(ed.pts); ts.append(np.zeros((len(ed.pts), d_out))); ms.append(np.zeros((len(ed.pts), d_out)))
            seg_n.append(len(ed.pts)); seg_normal.append(ed.normal); seg_edge.append(e)
            seg_start.append(pos); seg_sub.append(q)
            pos += len(ed.pts)
        n_res.append(len(s.x_f)); n_data.append(len(s.x_u))
        sub_off.append(pos); seg_off.append(len(seg_n))
        del parts
    n_points = pos
    # twins: local -> the neighbour's own segment of the same edge
    where = {(q, e): st for q, e, st in zip(seg_sub, seg_edge, seg_start)}
    send: Dict[int, List[int]] = {}
    recv_edges: Dict[int, List[Tuple[int, int, int]]] = {}
    for q, e, st, n in zip(seg_sub, seg_edge, seg_start, seg_n):
        nb = prob.edge_neighbor(q, e)
        if owner[nb] != owner[q]:
            peer = peer_of(owner[nb])
            send.setdefault(peer, []).append((e, q, st, n))
            recv_edges.setdefault(peer, []).append((e, nb, q, n))
    seg_twin = np.zeros(len(seg_n), dtype=np.int64)
    recv_rows: Dict[int, Tuple[int, int]] = {}
    row = n_points
    remote_slot = {}
    for peer in sorted(recv_edges):
        lst = sorted(recv_edges[peer])
        start = row
        for e, nb, q, n in lst:
            remote_slot[(q, e)] = row
            row += n
        recv_rows[peer] = (start, row - start)
    for i, (q, e, st) in enumerate(zip(seg_sub, seg_edge, seg_start)):
        nb = prob.edge_neighbor(q, e)
        seg_twin[i] = where[(nb, e)] if owner[nb] == owner[q] else remote_slot[(q, e)]
    send_idx = {}
    for peer, lst in send.items():
        idx = [np.arange(st, st + n) for e, q, st, n in sorted(lst)]
        send_idx[peer] = np.concatenate(idx).astype(np.int64)
    coords = np.concatenate(xs, axis=0).T.astype(np.float32) if n_points else np.zeros((2, 0), np.float32)
    target = np.concatenate(ts, axis=0).T.astype(np.float32) if n_points else np.zeros((d_out, 0), np.float32)
    mask = np.concatenate(ms, axis=0).T.astype(np.float32) if n_points else np.zeros((d_out, 0), np.float32)
    params = np.stack([prob.subdomains[q].params for q in local]).astype(np.float32)
    return PointTable(local, np.ascontiguousarray(coords), np.ascontiguousarray(target),
                      np.ascontiguousarray(mask), np.array(sub_off, np.int32), np.array(n_res, np.int32),
                      np.array(n_data, np.int32), np.array(seg_off, np.int32), np.array(seg_n, np.int32),
                      np.array(seg_normal, np.float32).reshape(-1, 2), seg_twin, np.array(seg_edge, np.int64),
                      params, ExchangePlan(send_idx, recv_rows, row - n_points))


def make_desc(prob, t: PointTable, dev_ptrs: Dict[str, int], stream: int = 0, flags: int = FLAG_GRAPH,
              hparams: Optional[Sequence] = None, norm_counts: Optional[Sequence] = None):
    """Fill a pinn_dd_desc; returns (desc, keep-alive list of host arrays)."""
    n_sub = len(t.local)
    if hparams is None:
        hparams = [(prob.w_u, prob.w_f, prob.w_i, prob.w_if, prob.lr, prob.beta1, prob.beta2, prob.eps)] * n_sub
    hp = (HParams * n_sub)(*[HParams(*map(float, h)) for h in hparams])
    keep = [hp]

    def ptr(a, ct):
        arr, p = _arr(a, ct)
        keep.append(arr)
        return p

    d = Desc()
    d.method, d.pde, d.activation = METHODS[prob.method], PDES[prob.pde], ACTS[prob.activation]
    d.d_in, d.d_out, d.width, d.n_hidden = 2, prob.d_out, prob.width, prob.n_hidden
    d.slope_n, d.nu, d.re = prob.slope_n, prob.nu, prob.re
    d.n_sub = n_sub
    d.sub_point_offset = ptr(t.sub_off, C.c_int32)
    d.sub_n_res = ptr(t.n_res, C.c_int32)
    d.sub_n_data = ptr(t.n_data, C.c_int32)
    d.sub_seg_offset = ptr(t.seg_off, C.c_int32)
    d.sub_hparams = C.cast(hp, C.POINTER(HParams))
    d.n_seg = len(t.seg_n)
    d.seg_n = ptr(t.seg_n if len(t.seg_n) else np.zeros(1, np.int32), C.c_int32)
    d.seg_normal = ptr(t.seg_normal.reshape(-1) if len(t.seg_n) else np.zeros(2, np.float32), C.c_float)
    d.seg_twin = ptr(t.seg_twin if len(t.seg_n) else np.zeros(1, np.int64), C.c_int64)
    d.n_points, d.n_recv = int(t.coords.shape[1]), t.plan.n_recv
    d.coords, d.target, d.mask = dev_ptrs.get("coords"), dev_ptrs.get("target"), dev_ptrs.get("mask")
    d.init_params = dev_ptrs.get("init_params")
    d.stream = stream
    d.flags = flags
    if norm_counts is not None:
        d.sub_norm_counts = ptr(np.asarray(norm_counts, dtype=np.int32).reshape(-1), C.c_int32)
    acts = [ACTS[prob.act(q)] for q in t.local]
    if any(a != d.activation for a in acts):
        d.sub_activation = ptr(np.asarray(acts, dtype=np.int32), C.c_int32)
    # exchange plan (peers ascending; received ranges in the same order)
    peers = sorted(set(t.plan.send) | set(t.plan.recv))
    if peers:
        sends = [np.asarray(t.plan.send.get(p, np.zeros(0, np.int64)), np.int64) for p in peers]
        off = np.concatenate([[0], np.cumsum([len(x) for x in sends])]).astype(np.int64)
        d.n_peers = len(peers)
        d.peer_rank = ptr(np.asarray(peers, np.int32), C.c_int32)
        d.peer_send_off = ptr(off, C.c_int64)
        d.send_rows = ptr(np.concatenate(sends) if off[-1] else np.zeros(1, np.int64), C.c_int64)
        row = int(t.coords.shape[1])
        rr, rn = [], []
        for p in peers:
            r0, n = t.plan.recv.get(p, (row, 0))
            rr.append(r0)
            rn.append(n)
            row = r0 + n
        d.peer_recv_row = ptr(np.asarray(rr, np.int64), C.c_int64)
        d.peer_recv_n = ptr(np.asarray(rn, np.int64), C.c_int64)
    # Eq. (4) geometry of the whole decomposition
    pos = {q: i for i, q in enumerate(t.local)}
    d.geo_local = ptr(np.asarray([pos.get(q, -1) for q in range(prob.n_sub)], np.int32), C.c_int32)
    d.n_geo = prob.n_sub
    if "seeds" in prob.meta:
        d.geometry = GEOM_VORONOI
        d.geo = ptr(np.asarray(prob.meta["seeds"], np.float32).reshape(-1), C.c_float)
        poly = np.asarray(prob.meta["polygon"], np.float32)
        d.n_poly = len(poly)
        d.poly = ptr(poly.reshape(-1), C.c_float)
        d.geo_tol = 1e-5
    else:
        d.geometry = GEOM_BOXES
        d.geo = ptr(np.asarray([[s.lo[0], s.lo[1], s.hi[0], s.hi[1]] for s in prob.subdomains],
                               np.float32).reshape(-1), C.c_float)
        d.geo_tol = 0.0
    return d, keep


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId from the library's NCCL (pinn_dd_nccl_unique_id)."""
    lib = load_library()
    buf = (C.c_char * 128)()
    st = lib.pinn_dd_nccl_unique_id(buf)
    if st != OK:
        raise PinnDDError(st, lib.pinn_dd_last_error(None).decode())
    return bytes(buf)


class PinnDD:
    """One handle per GPU: the subdomains `local` of `prob`.

    transport="nccl": cut-edge payload rows move inside the library (NCCL P2P
    on an internal stream, captured with the rest of the iteration into one
    CUDA graph by pinn_dd_step).  With world > 1, rank 0 draws the NCCL id and
    `group` (a torch.distributed process group, any backend) broadcasts it.
    transport="peer": the rows are stored straight into the neighbours' memory
    by the fused launch (CUDA IPC handles traded over `group`).
    loopback=True (single process): edges between different owners are
    exchanged with this rank itself through the chosen transport -- the
    multi-GPU data path validated on one GPU."""

    def __init__(self, prob, local: Optional[Sequence[int]] = None, owner: Optional[Sequence[int]] = None,
                 rank: int = 0, device=None, flags: int = FLAG_GRAPH, hparams: Optional[Sequence] = None,
                 norm_counts: Optional[Sequence] = None, transport: Optional[str] = None, world: int = 1,
                 group=None, loopback: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("PinnDD needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.prob = prob
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        local = list(range(prob.n_sub)) if local is None else list(local)
        self.table = build_point_table(prob, local, owner, rank, peer_of=(lambda o: rank) if loopback else None)
        t = self.table
        dev = self.device
        self.n_sub = len(local)
        self.n_params = int(self.lib.pinn_dd_n_params(2, prob.width, prob.n_hidden, prob.d_out))
        assert self.n_params == t.params.shape[1]
        # device point table (borrowed by the library until destroy)
        self.coords = torch.from_numpy(t.coords).to(dev)
        self.target = torch.from_numpy(t.target).to(dev)
        self.mask = torch.from_numpy(t.mask).to(dev)
        self.init_params = torch.from_numpy(t.params).to(dev)
        self.n_points = int(t.coords.shape[1])
        self.stream = torch.cuda.current_stream(dev)
        d, self._keep = make_desc(prob, t, dict(coords=self.coords.data_ptr(), target=self.target.data_ptr(),
                                               mask=self.mask.data_ptr(), init_params=self.init_params.data_ptr()),
                                  self.stream.cuda_stream, flags, hparams, norm_counts)
        nccl_id = None
        if transport == "peer":
            flags |= FLAG_PEER_STORES
            d.flags = flags
            d.rank, d.world = (rank, 1) if loopback else (rank, world)
        elif transport == "nccl":
            if world > 1:
                import torch.distributed as dist
                obj = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                nccl_id = obj[0]
            else:
                nccl_id = nccl_unique_id()
            self._nccl_id = C.create_string_buffer(nccl_id, 128)
            d.nccl_id = C.cast(self._nccl_id, C.c_void_p)
            d.rank, d.world = (0, 1) if loopback else (rank, world)
        elif transport is not None:
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        self.rank = rank
        self.desc = d
        nbytes = C.c_size_t(0)
        self._check(self.lib.pinn_dd_workspace_size(C.byref(d), C.byref(nbytes)), None)
        self.workspace = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=dev)
        h = C.c_void_p()
        self._check(self.lib.pinn_dd_create(C.byref(d), C.c_void_p(self.workspace.data_ptr()),
                                            nbytes.value, C.byref(h)), None)
        self.h = h
        buf, nf, nrows = C.c_void_p(), C.c_int32(), C.c_int64()
        self._check(self.lib.pinn_dd_payload_buffer(self.h, C.byref(buf), C.byref(nf), C.byref(nrows)))
        self.n_fields, self.n_rows, self._payload_ptr = nf.value, nrows.value, buf.value
        off = self._payload_ptr - self.workspace.data_ptr()
        assert off % 4 == 0
        self.payload = self.workspace[off: off + 4 * self.n_rows * self.n_fields].view(torch.float32).view(
            self.n_rows, self.n_fields)
        if transport == "peer":
            self._connect_peers(group, world, loopback)

    def _connect_peers(self, group, world, loopback):
        """Trade the exchange regions (CUDA IPC) and connect every peer of the plan."""
        handle = (C.c_char * 64)()
        foff, roff = C.c_int64(), C.c_int64()
        self._check(self.lib.pinn_dd_ipc_export(self.h, handle, C.byref(foff), C.byref(roff)))
        plan = self.table.plan
        peers = sorted(set(plan.send) | set(plan.recv))
        mine = dict(rank=self.rank, handle=bytes(handle), foff=foff.value, roff=roff.value, peers=peers,
                    recv={p: plan.recv.get(p, (0, 0))[0] for p in peers}, n_recv=plan.n_recv)
        if loopback or world == 1:
            allinfo = {self.rank: mine}
        else:
            import torch.distributed as dist
            got = [None] * world
            dist.all_gather_object(got, mine, group=group)
            allinfo = {g["rank"]: g for g in got}
        n = len(peers)
        hs = (C.c_char * (64 * max(1, n)))()
        fo, ro, prow, pn = (C.c_int64 * max(1, n))(), (C.c_int64 * max(1, n))(), (C.c_int64 * max(1, n))(), \
            (C.c_int64 * max(1, n))()
        pf = (C.c_int32 * max(1, n))()
        for i, p in enumerate(peers):
            o = allinfo[p]
            C.memmove(C.addressof(hs) + 64 * i, o["handle"], 64)
            fo[i], ro[i] = o["foff"], o["roff"]
            prow[i] = o["recv"][self.rank]
            pn[i] = o["n_recv"]
            pf[i] = o["peers"].index(self.rank)
        st = self.lib.pinn_dd_connect_peers(self.h, hs, fo, ro, prow, pn, pf)
        if not (loopback or world == 1):
            # every rank connected, or every rank raises (no rank left waiting in a step)
            import torch.distributed as dist
            dev = self.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
            ok = torch.tensor([1 if st == OK else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if st == OK and int(ok.item()) == 0:
                raise PinnDDError(EPROTOCOL, "peer stores: another rank failed to connect")
        self._check(st)

    # ------------------------------------------------------------------
    def _check(self, status, h="self"):
        if status != OK:
            hh = self.h if (h == "self" and getattr(self, "h", None)) else None
            msg = self.lib.pinn_dd_last_error(hh)
            raise PinnDDError(status, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "h", None):
            self.lib.pinn_dd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI
    def interface_payload(self):
        self._check(self.lib.pinn_dd_interface_payload(self.h))

    def loss_grad(self, want_grad: bool = True):
        loss = torch.empty(self.n_sub, 8, dtype=torch.float32, device=self.device)
        grad = torch.empty(self.n_sub, self.n_params, dtype=torch.float32, device=self.device) if want_grad else None
        self._check(self.lib.pinn_dd_loss_grad(self.h, C.c_void_p(loss.data_ptr()),
                                               C.c_void_p(grad.data_ptr()) if want_grad else None))
        return loss, grad

    def adam(self):
        self._check(self.lib.pinn_dd_adam(self.h))

    def step(self, n_iters: int = 1, want_loss: bool = True):
        out = np.zeros((self.n_sub, 8), dtype=np.float32) if want_loss else None
        p = out.ctypes.data_as(C.POINTER(C.c_float)) if want_loss else None
        self._check(self.lib.pinn_dd_step(self.h, int(n_iters), p))
        return out

    def loss_grad_phased(self, exchange=None, want_grad: bool = True):
        """pinn_dd_loss_grad in two halves: K1 over residual + training points,
        then `exchange()` (if given; e.g. waits for the payload receives), then K1
        over interface points + K5a.  Same results as loss_grad, bit for bit."""
        loss = torch.empty(self.n_sub, 8, dtype=torch.float32, device=self.device)
        grad = torch.empty(self.n_sub, self.n_params, dtype=torch.float32, device=self.device) if want_grad else None
        self._check(self.lib.pinn_dd_loss_grad_interior(self.h))
        if exchange is not None:
            exchange()
        self._check(self.lib.pinn_dd_loss_grad_interface(self.h, C.c_void_p(loss.data_ptr()),
                                                         C.c_void_p(grad.data_ptr()) if want_grad else None))
        return loss, grad

    def step_distributed(self, n_iters: int = 1, group=None, want_loss: bool = False):
        """Algorithm 1 with remote neighbours: payload (K2) ->
        non-blocking exchange with the neighbouring ranks, overlapped with K1 over
        the residual and training points -> wait -> K1 over the interface points
        and K5a -> Adam (K5b).  Returns the last iteration's [n_sub, 8] loss
        breakdown (host) if want_loss."""
        if not hasattr(self, "_loss_dev"):
            self._loss_dev = torch.empty(self.n_sub, 8, dtype=torch.float32, device=self.device)
        for _ in range(n_iters):
            self.interface_payload()
            reqs = exchange_payload(self.payload, self.table.plan, group, wait=False)
            self._check(self.lib.pinn_dd_loss_grad_interior(self.h))
            for r in reqs:
                r.wait()
            self._check(self.lib.pinn_dd_loss_grad_interface(self.h, C.c_void_p(self._loss_dev.data_ptr()),
                                                             None))
            self.adam()
        return self._loss_dev.cpu().numpy() if want_loss else None

    def predict(self, pts: torch.Tensor, owners: Optional[torch.Tensor] = None, mode: str = "stitched") -> torch.Tensor:
        """Eq. (4): pts [2, n] float32 -> [d_out, n].  Owners classified by the
        library from the decomposition's geometry (mode "stitched": 1/S
        average; "owner": lowest-id owner), or the caller's owners [n, 4] int32
        local ids (-1 unused).  With several ranks each returns its local
        owners' share (sum over ranks)."""
        n = pts.shape[1]
        out = torch.empty(self.prob.d_out, n, dtype=torch.float32, device=self.device)
        pts = pts.contiguous()
        if owners is not None:
            owners = owners.contiguous()
            self._check(self.lib.pinn_dd_predict_owners(self.h, C.c_void_p(pts.data_ptr()),
                                                        C.c_void_p(owners.data_ptr()), n, C.c_void_p(out.data_ptr())))
        else:
            m = {"stitched": PREDICT_STITCHED, "owner": PREDICT_OWNER}[mode]
            self._check(self.lib.pinn_dd_predict(self.h, C.c_void_p(pts.data_ptr()), n, C.c_void_p(out.data_ptr()), m))
        return out

    def exchange(self):
        """The library's NCCL exchange of the cut-edge payload rows (phased path)."""
        self._check(self.lib.pinn_dd_exchange(self.h))

    def get(self, q: int, what: int = 0) -> torch.Tensor:
        out = torch.empty(self.n_params, dtype=torch.float32, device=self.device)
        self._check(self.lib.pinn_dd_get_params(self.h, q, what, C.c_void_p(out.data_ptr())))
        return out

    def set(self, q: int, values: torch.Tensor, what: int = 0):
        v = values.to(self.device, torch.float32).contiguous()
        self._check(self.lib.pinn_dd_set_params(self.h, q, what, C.c_void_p(v.data_ptr())))

    def adam_t(self, q: int) -> int:
        t = C.c_int32()
        self._check(self.lib.pinn_dd_get_step(self.h, q, C.byref(t)))
        return t.value

    def read_loss(self, dst: torch.Tensor):
        """Enqueue the copy of the last [n_sub, 8] loss breakdown into dst (pinned
        host or device tensor) on the handle's stream; no synchronisation."""
        assert dst.dtype == torch.float32 and dst.is_contiguous() and dst.numel() >= self.n_sub * 8
        self._check(self.lib.pinn_dd_read_loss(self.h, C.c_void_p(dst.data_ptr())))

    @property
    def step_fused(self) -> bool:
        """pinn_dd_step runs K2 (payload) inside K1's persistent launch."""
        return bool(self.lib.pinn_dd_step_fused(self.h))

    def kernel_times(self):
        """[K2, K1, K5, launches, exchange, K1 interior, K1 interface, exposed exchange wait] (ms)."""
        ms = (C.c_double * 8)()
        self._check(self.lib.pinn_dd_kernel_times(self.h, ms))
        return list(ms)

    def debug_buffer(self, which: int, dtype=torch.int32) -> torch.Tensor:
        """Copy of an internal device buffer (tests / debugging)."""
        ptr, nb = C.c_void_p(), C.c_int64()
        self._check(self.lib.pinn_dd_debug_buffer(self.h, which, C.byref(ptr), C.byref(nb)))
        off = ptr.value - self.workspace.data_ptr()
        return self.workspace[off: off + nb.value].view(dtype).clone()

    def plan_info(self):
        v = (C.c_int64 * 4)()
        self._check(self.lib.pinn_dd_plan_info(self.h, v))
        return list(v)


def exchange_payload(payload: torch.Tensor, plan: ExchangePlan, group=None, wait: bool = True):
    """Green stage of Algorithm 1: non-blocking send/recv of the cut-edge payload
    rows with every neighbouring rank; waits unless
    wait=False, in which case the request handles are returned (NCCL: waiting
    makes the current stream wait, so interior compute enqueued before it
    overlaps the transfer).  Works on CUDA tensors with NCCL and on CPU tensors
    with gloo."""
    import torch.distributed as dist
    if not plan.send and not plan.recv:
        return []
    # gloo moves host memory only: CUDA payload rows are staged through the host
    # (test / CPU-cluster path; NCCL sends the device rows directly)
    stage = payload.is_cuda and dist.get_backend(group) == "gloo"
    ops, bufs, landing = [], [], []
    cache = plan.__dict__.setdefault("_idx_cache", {})
    for peer in sorted(set(plan.send) | set(plan.recv)):
        if peer in plan.send:
            key = (peer, str(payload.device))
            if key not in cache:
                cache[key] = torch.as_tensor(plan.send[peer], device=payload.device)
            idx = cache[key]
            sbuf = payload.index_select(0, idx).contiguous()
            if stage:
                sbuf = sbuf.cpu()
            bufs.append(sbuf)
            ops.append(dist.P2POp(dist.isend, sbuf, peer, group))
        if peer in plan.recv:
            r0, n = plan.recv[peer]
            if stage:
                rbuf = torch.empty(n, payload.shape[1], dtype=payload.dtype)
                landing.append((r0, n, rbuf))
            else:
                rbuf = payload[r0:r0 + n]
            ops.append(dist.P2POp(dist.irecv, rbuf, peer, group))
    reqs = dist.batch_isend_irecv(ops)
    if wait or stage:
        for req in reqs:
            req.wait()
        for r0, n, rbuf in landing:
            payload[r0:r0 + n].copy_(rbuf)
        return []
    return reqs


# ---------------------------------------------------------------------------
# Data-parallel vanilla PINN (the paper's comparator, Fig. 1a / Table 2,
# PAPER.md:38, 55, 737-768): one network replicated on every rank, the point
# sets sharded, gradients summed with an all-reduce, identical Adam steps.
# ---------------------------------------------------------------------------

def shard_problem(prob, rank: int, world: int):
    """Rank `rank`'s share (every world-th point) of a single-subdomain problem,
    and the full-data counts (N_F, N_u) used for its 1/N normalisation."""
    import dataclasses
    if prob.n_sub != 1:
        raise ValueError("data-parallel PINN shards a single network / subdomain")
    s = prob.subdomains[0]
    s2 = dataclasses.replace(s, x_f=s.x_f[rank::world], x_u=s.x_u[rank::world],
                             u_target=s.u_target[rank::world], u_mask=s.u_mask[rank::world])
    return dataclasses.replace(prob, subdomains=[s2]), (len(s.x_f), len(s.x_u))


class DataParallelPINN:
    """Each rank: loss + gradient of its shard (K1, K5a) -> all-reduce(sum) of the
    gradient and loss breakdown -> Adam (K5b) on the summed gradient."""

    def __init__(self, prob, rank: int = 0, world: int = 1, device=None, group=None, flags: int = 0):
        shard, counts = shard_problem(prob, rank, world)
        self.world, self.group = world, group
        self.h = PinnDD(shard, device=device, flags=flags, norm_counts=[counts])

    def step(self, n_iters: int = 1, want_loss: bool = False):
        import torch.distributed as dist
        loss = None
        for _ in range(n_iters):
            loss, grad = self.h.loss_grad()
            if self.world > 1:
                dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
                dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=self.group)
            self.h.set(0, grad[0], what=3)
            self.h.adam()
        return loss.cpu().numpy() if want_loss else None

    def close(self):
        self.h.close()
