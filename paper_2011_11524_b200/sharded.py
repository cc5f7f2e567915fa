"""One large product sharded over G GPUs (configs 4 and 5).

The transform of length N runs its first K passes column-sharded (rank q owns columns
[q Bc, (q + 1) Bc) of the Rtot x Sc pass matrix) and the rest row-sharded (rank q owns
Rtot / G whole segments of length Sc); one all-to-all per direction moves between the
two layouts — the six-step transposition done over NVLink. A last all-to-all leaves rank
q with the natural-order coefficients [q N / G, (q + 1) N / G), whose carries are resolved
with an all-gather of per-rank {0,1,2}-carry maps (a few bytes per rank).

Per product and per prime: 4 all-to-alls of N / G words per rank (x forward, y forward,
inverse, natural redistribution) — 3 when squaring.

The device steps live in libdecmul_gpu.so (``decmul_gpu_shard_*``); this module only
sequences them and moves buffers. Transports (``Comm``):

* ``TorchComm`` — torch.distributed (NCCL between GPUs; gloo in CPU tests);
* ``LocalComm`` — all G shards in one process on one device, exchanged by copies
  (sequential, so no shard ever waits on another — safe on a single GPU).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _raise, load_library

COL_FWD, ROW_FWD, ROW_FWD_CONV, COL_INV = 0, 1, 2, 3
IDENTITY_MAP = 0x24


class ShardPlan(C.Structure):
    _fields_ = [("length", C.c_size_t), ("base_exp", C.c_uint), ("p1", C.c_uint64), ("p2", C.c_uint64),
                ("ranks", C.c_int), ("col_passes", C.c_int), ("rows", C.c_size_t), ("seg_len", C.c_size_t),
                ("col_width", C.c_size_t), ("local_len", C.c_size_t), ("s_words", C.c_size_t),
                ("map_words", C.c_size_t), ("digits_x", C.c_size_t), ("digits_y", C.c_size_t),
                ("top_candidates", C.c_ulonglong * 2)]


# ---- {0,1,2}-carry maps (same encoding as csrc/carry.cuh) ----

def map_apply(m: int, c: int) -> int:
    return (m >> (2 * c)) & 3


def map_compose(later: int, earlier: int) -> int:
    return sum(map_apply(later, map_apply(earlier, c)) << (2 * c) for c in range(3))


def rank_carry_ins(rank_maps: list[int]) -> list[int]:
    """Carry into each rank: the composed maps of all earlier ranks applied to 0."""
    out, acc = [], IDENTITY_MAP
    for m in rank_maps:
        out.append(map_apply(acc, 0))
        acc = map_compose(m, acc)
    return out


def decimal_len(v: int) -> int:
    return len(str(v))


def rank_digit_range(plan, q: int, n: int) -> tuple[int, int]:
    """Bytes [lo, hi) of the n-digit product text written by shard q (its limbs
    [q L, (q + 1) L) are one contiguous digit range; the top limb is unpadded)."""
    be, L = int(plan.base_exp), int(plan.local_len)
    top = (n - 1) // be
    top_len = n - top * be
    k_lo, k_hi = q * L, min((q + 1) * L - 1, top)
    if k_lo > top:
        return n, n

    def pos(k):
        return 0 if k == top else top_len + (top - 1 - k) * be

    return pos(k_hi), pos(k_lo) + (top_len if k_lo == top else be)


# ---- transports ----

class LocalComm:
    """All ranks are local shards of one process (one device); exchanges are copies."""

    def __init__(self, G: int):
        self.G = G

    def all_to_all(self, sends, recvs):
        G = self.G
        n = sends[0].numel() // G
        for d in range(G):
            for s in range(G):
                recvs[d][s * n:(s + 1) * n].copy_(sends[s][d * n:(d + 1) * n])

    def all_gather(self, values):
        return list(values)


class TorchComm:
    """One shard per process over torch.distributed (NCCL for CUDA tensors, gloo for CPU).
    The carry protocol's small all-gathers (halo residues, carry maps, top-limb probes)
    go as int64 tensors — on the GPU under NCCL — rather than pickled objects."""

    def __init__(self, dist):
        import torch

        self.dist = dist
        self.torch = torch
        self.G = dist.get_world_size()
        nccl = dist.get_backend() == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def all_to_all(self, sends, recvs):
        (send,), (recv,) = sends, recvs
        self.dist.all_to_all_single(recv, send)

    def all_gather(self, values):
        (v,) = values
        t = self.torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.uint64)).view(np.int64)).to(self.device)
        out = [self.torch.empty_like(t) for _ in range(self.G)]
        self.dist.all_gather(out, t)
        return [o.cpu().numpy().view(np.uint64) for o in out]


# ---- device backend (libdecmul_gpu.so on torch CUDA tensors) ----

class DeviceBackend:
    """Library calls and the torch-side copies/exchanges share ONE stream (the library
    otherwise uses its context's non-blocking stream, unordered with torch's)."""

    def __init__(self, ctx, stream=None):
        import torch

        self.torch = torch
        self.ctx = ctx
        self.device = torch.device("cuda", ctx.device)
        self.stream_obj = stream if stream is not None else torch.cuda.Stream(self.device)
        self.stream = self.stream_obj.cuda_stream
        load_library()

    def scope(self):
        return self.torch.cuda.stream(self.stream_obj)

    def _p(self, t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def plan(self, nx: int, ny: int, G: int) -> ShardPlan:
        p = ShardPlan()
        self.ctx._call("decmul_gpu_shard_plan_create", C.c_size_t(nx), C.c_size_t(ny), C.c_int(G), C.byref(p))
        return p

    def zeros(self, n: int):
        return self.torch.zeros(n, dtype=self.torch.int64, device=self.device)

    def pack(self, plan, q, digits, nd, out):
        self.ctx._call("decmul_gpu_shard_pack", C.byref(plan), C.c_int(q), C.c_void_p(digits.data_ptr()),
                       C.c_size_t(nd), self._p(out), C.c_void_p(self.stream))

    def transform(self, plan, q, stage, src, dst, other=None):
        o = other or (None, None)
        self.ctx._call("decmul_gpu_shard_transform", C.byref(plan), C.c_int(q), C.c_int(stage), self._p(src[0]),
                       self._p(src[1]), self._p(dst[0]), self._p(dst[1]), self._p(o[0]), self._p(o[1]),
                       C.c_void_p(self.stream))

    def reorder(self, plan, to_segments, src, dst):
        self.ctx._call("decmul_gpu_shard_reorder", C.byref(plan), C.c_int(int(to_segments)), self._p(src),
                       self._p(dst), C.c_void_p(self.stream))

    def last_two(self, z):
        return np.concatenate([z[0][-2:].cpu().numpy().view(np.uint64), z[1][-2:].cpu().numpy().view(np.uint64)])

    def carry_begin(self, plan, q, z, halo, s, maps) -> int:
        h = (C.c_uint64 * 4)(*[int(v) for v in halo])
        rm = C.c_uint()
        self.ctx._call("decmul_gpu_shard_carry_begin", C.byref(plan), C.c_int(q), self._p(z[0]), self._p(z[1]), h,
                       self._p(s), self._p(maps), C.byref(rm), C.c_void_p(self.stream))
        return rm.value

    def carry_probe(self, plan, q, cin, z, s, maps):
        zo = (C.c_uint64 * 2)()
        self.ctx._call("decmul_gpu_shard_carry_probe", C.byref(plan), C.c_int(q), C.c_uint(cin), self._p(z[0]),
                       self._p(z[1]), self._p(s), self._p(maps), zo, C.c_void_p(self.stream))
        return [zo[0], zo[1]]

    def carry_emit(self, plan, q, cin, top, top_len, z, s, maps, out):
        self.ctx._call("decmul_gpu_shard_carry_emit", C.byref(plan), C.c_int(q), C.c_uint(cin), C.c_ulonglong(top),
                       C.c_uint(top_len), self._p(z[0]), self._p(z[1]), self._p(s), self._p(maps),
                       C.c_void_p(out.data_ptr()), C.c_void_p(self.stream))


# ---- the product ----

def sharded_multiply(backend, comm, plan, shards, xs, ys, outs, squaring=False) -> int:
    """Multiply on the local `shards` (rank ids) of a G-rank job.

    xs[i], ys[i]: operand digits visible to shard shards[i] (full strings);
    outs[i]: a full-length output buffer; shard q writes its limbs' digits at their
    global positions. Returns the product length (same on every rank)."""
    with backend.scope():
        return _sharded_multiply(backend, comm, plan, shards, xs, ys, outs, squaring)


def _sharded_multiply(backend, comm, plan, shards, xs, ys, outs, squaring):
    L = int(plan.local_len)
    st = {q: dict(X=[backend.zeros(L), backend.zeros(L)], Y=[backend.zeros(L), backend.zeros(L)],
                  P=backend.zeros(L), R=backend.zeros(L), S=backend.zeros(int(plan.s_words)),
                  M=backend.zeros(int(plan.map_words))) for q in shards}

    def to_segments(key):  # column layout -> all-to-all -> contiguous segments
        for pr in (0, 1):
            comm.all_to_all([st[q][key][pr] for q in shards], [st[q]["R"] for q in shards])
            for q in shards:
                backend.reorder(plan, True, st[q]["R"], st[q][key][pr])

    def to_columns(key):  # segments -> blocks -> all-to-all -> column layout
        for pr in (0, 1):
            for q in shards:
                backend.reorder(plan, False, st[q][key][pr], st[q]["R"])
            comm.all_to_all([st[q]["R"] for q in shards], [st[q][key][pr] for q in shards])

    nx, ny = int(plan.digits_x), int(plan.digits_y)
    for i, q in enumerate(shards):
        backend.pack(plan, q, xs[i], nx, st[q]["P"])
        backend.transform(plan, q, COL_FWD, (st[q]["P"], st[q]["P"]), st[q]["X"])
    to_segments("X")
    if squaring:
        key = "X"
        for q in shards:
            backend.transform(plan, q, ROW_FWD_CONV, st[q]["X"], st[q]["X"], None)
    else:
        key = "Y"
        for i, q in enumerate(shards):
            backend.transform(plan, q, ROW_FWD, st[q]["X"], st[q]["X"])
            backend.pack(plan, q, ys[i], ny, st[q]["P"])
            backend.transform(plan, q, COL_FWD, (st[q]["P"], st[q]["P"]), st[q]["Y"])
        to_segments("Y")
        for q in shards:
            backend.transform(plan, q, ROW_FWD_CONV, st[q]["Y"], st[q]["Y"], st[q]["X"])
    to_columns(key)
    for q in shards:
        backend.transform(plan, q, COL_INV, st[q][key], st[q][key])
    to_segments(key)  # rank q now holds coefficients [q N / G, (q + 1) N / G) in natural order
    # ---- distributed carry ----
    lasts = comm.all_gather([backend.last_two(st[q][key]) for q in shards])
    rmaps_local = []
    for q in shards:
        halo = np.zeros(4, np.uint64) if q == 0 else np.asarray(lasts[q - 1], np.uint64)
        rmaps_local.append(np.array([backend.carry_begin(plan, q, st[q][key], halo, st[q]["S"], st[q]["M"])],
                                    np.uint64))
    rmaps = [int(v[0]) for v in comm.all_gather(rmaps_local)]
    cins = rank_carry_ins(rmaps)
    probes = comm.all_gather([np.array(backend.carry_probe(plan, q, cins[q], st[q][key], st[q]["S"], st[q]["M"]),
                                       np.uint64) for q in shards])
    none = np.uint64(2**64 - 1)
    zc = [next((int(p[t]) for p in probes if p[t] != none), 0) for t in (0, 1)]
    cand = [int(plan.top_candidates[0]), int(plan.top_candidates[1])]
    if zc[1] != 0:
        top, z = cand[1], zc[1]
    elif zc[0] != 0:
        top, z = cand[0], zc[0]
    else:
        top, z = 0, 0
    top_len = decimal_len(z)
    for i, q in enumerate(shards):
        backend.carry_emit(plan, q, cins[q], top, top_len, st[q][key], st[q]["S"], st[q]["M"], outs[i])
    return top_len + top * int(plan.base_exp)
