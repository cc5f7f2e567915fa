"""TEST INFRASTRUCTURE: a CPU emulation of the sharded device steps (decmul_gpu_shard_*),
so the multi-rank driver (paper_2011_11524_b200/sharded.py) — its layouts, all-to-all
chunking, block reorders and distributed carry protocol — runs over gloo on CPU.

Each step restates the math of the corresponding kernel on Python ints:
pass i forward = length-R column DFTs of stride S with outputs at bit-reversed
positions, then the twiddle omega_{R S}^{f s} (kernels.cu k_pass_fwd, k_radix3_fwd);
inverse = conjugate twiddle (times the convolution scale on the last table pass) then
unscaled inverse DFT; the fused last pass = DIF, REDC pointwise, DIT. Column-phase
passes use the global column ((s >> cb) << sb) + q Bc + (s mod Bc) for their twiddle.
Planning comes from the real library (decmul_gpu_shard_plan_create with no context).
Never used by the product path.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np
import torch

import oracle
import paper_2011_11524_b200 as dm
from paper_2011_11524_b200.sharded import COL_FWD, COL_INV, ROW_FWD, ROW_FWD_CONV, ShardPlan, map_apply, map_compose

R64 = 1 << 64


def _bitrev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


class EmuBackend:
    def __init__(self):
        self.port = oracle.port()
        self._carry = {}

    def scope(self):
        return contextlib.nullcontext()

    def plan(self, nx, ny, G) -> ShardPlan:
        p = ShardPlan()
        rc = dm.load_library().decmul_gpu_shard_plan_create(None, C.c_size_t(nx), C.c_size_t(ny), C.c_int(G),
                                                           C.byref(p))
        if rc:
            raise ValueError("shard plan failed")
        N = p.length
        rad = [3] if N % 3 == 0 else []
        c = N // 3 if rad else N
        k = c.bit_length() - 1
        m = -(-k // 9)
        rad += [1 << (k // m + (1 if i < k % m else 0)) for i in range(m)]
        self.radices = rad
        return p

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.int64)

    # ---- steps ----
    def pack(self, plan, q, digits, nd, out):
        be, Bc, Sc = plan.base_exp, plan.col_width, plan.seg_len
        s = bytes(digits)
        nl = -(-nd // be)
        vals = []
        for i in range(plan.local_len):
            t = (i // Bc) * Sc + q * Bc + (i % Bc)
            if t < nl:
                end = nd - t * be
                vals.append(int(s[max(0, end - be):end]))
            else:
                vals.append(0)
        out.copy_(torch.tensor(vals, dtype=torch.int64))

    def _field(self, plan, pr):
        p = plan.p1 if pr == 0 else plan.p2
        N = plan.length
        xi = self.port.primitive_root(p, N)
        return p, N, xi

    def _geom(self, plan, i, q, sharded_cols):
        """(R, S_local, groups, colmap) of pass i on this rank's array."""
        N, G = plan.length, plan.ranks
        R = self.radices[i]
        S = N // int(np.prod(self.radices[: i + 1]))
        if sharded_cols:
            Sl = S // G
            cb, sb = plan.col_width.bit_length() - 1, plan.seg_len.bit_length() - 1
            off = q * plan.col_width
            colmap = lambda s: ((s >> cb) << sb) + off + (s & (plan.col_width - 1))  # noqa: E731
            groups = N // (R * S)
        else:
            Sl, colmap, groups = S, (lambda s: s), N // (R * S) // G
        return R, S, Sl, groups, colmap

    def _last_table(self, plan):
        N = plan.length
        lt = -1
        for i, R in enumerate(self.radices):
            S = N // int(np.prod(self.radices[: i + 1]))
            if R == 3 or S > 1:
                lt = i
        return lt

    @staticmethod
    def _powers(w, n, p):
        out, acc = [], 1
        for _ in range(n):
            out.append(acc)
            acc = acc * w % p
        return out

    def _dft(self, v, wpow, p):
        R = len(v)
        return [sum(v[r] * wpow[r * f % R] for r in range(R)) % p for f in range(R)]

    def _pass(self, a, plan, pr, i, q, sharded_cols, inverse):
        p, N, xi = self._field(plan, pr)
        R, S, Sl, groups, colmap = self._geom(plan, i, q, sharded_cols)
        M = R * S
        wM = pow(xi, N // M, p)
        wR = pow(xi, N // R, p)
        if inverse:
            wM, wR = pow(wM, p - 2, p), pow(wR, p - 2, p)
        wpow = self._powers(wR, R, p)
        tw = self._powers(wM, M, p)
        scale = (R64 % p) * pow(N % p, p - 2, p) % p if (inverse and i == self._last_table(plan)) else 1
        bits = (R.bit_length() - 1) if R != 3 else 0
        pos_of = [_bitrev(f, bits) for f in range(R)] if R != 3 else [0, 1, 2]  # spectrum f -> position
        for g in range(groups):
            for s in range(Sl):
                idx = [g * R * Sl + r * Sl + s for r in range(R)]
                sg = colmap(s)
                if not inverse:
                    spec = self._dft([a[j] for j in idx], wpow, p)
                    for f in range(R):
                        a[idx[pos_of[f]]] = spec[f] * tw[f * sg % M] % p
                else:
                    yf = [a[idx[pos_of[f]]] * tw[f * sg % M] * scale % p for f in range(R)]
                    for j, val in zip(idx, self._dft(yf, wpow, p)):
                        a[j] = val

    def _fused(self, a, plan, pr, q, other):
        """Last pass (S == 1): DIF, pointwise REDC (a b R^-1) against `other`, DIT."""
        p, N, xi = self._field(plan, pr)
        R, _, _, groups, _ = self._geom(plan, len(self.radices) - 1, q, False)
        wR = pow(xi, N // R, p)
        fwd, inv = self._powers(wR, R, p), self._powers(pow(wR, p - 2, p), R, p)
        rinv = pow(R64 % p, p - 2, p)
        bits = R.bit_length() - 1
        pos_of = [_bitrev(f, bits) for f in range(R)]
        for g in range(groups):
            idx = [g * R + r for r in range(R)]
            spec = self._dft([a[j] for j in idx], fwd, p)
            o = spec if other is None else [other[idx[pos_of[f]]] for f in range(R)]
            prod = [spec[f] * o[f] % p * rinv % p for f in range(R)]
            for j, val in zip(idx, self._dft(prod, inv, p)):
                a[j] = val

    def transform(self, plan, q, stage, src, dst, other=None):
        K, m = plan.col_passes, len(self.radices)
        for pr in (0, 1):
            a = [int(v) for v in src[pr].tolist()]
            if stage == COL_FWD:
                for i in range(K):
                    self._pass(a, plan, pr, i, q, True, False)
            elif stage == ROW_FWD:
                for i in range(K, m):
                    self._pass(a, plan, pr, i, q, False, False)
            elif stage == ROW_FWD_CONV:
                for i in range(K, m - 1):
                    self._pass(a, plan, pr, i, q, False, False)
                o = None if other is None else [int(v) for v in other[pr].tolist()]
                self._fused(a, plan, pr, q, o)
                for i in reversed(range(K, m - 1)):
                    self._pass(a, plan, pr, i, q, False, True)
            elif stage == COL_INV:
                for i in reversed(range(K)):
                    self._pass(a, plan, pr, i, q, True, True)
            dst[pr].copy_(torch.tensor(a, dtype=torch.int64))

    def reorder(self, plan, to_segments, src, dst):
        G, rows, w = plan.ranks, plan.rows // plan.ranks, plan.col_width
        x = src.view(G, rows, w) if to_segments else src.view(rows, G, w)
        dst.copy_(x.transpose(0, 1).reshape(-1))

    def last_two(self, z):
        return np.array([int(z[0][-2]), int(z[0][-1]), int(z[1][-2]), int(z[1][-1])], dtype=np.uint64)

    # ---- carry (decimal.cpp:154-189 restated over this rank's block) ----
    def _limbs(self, plan, q, z, halo):
        p1, p2, be = plan.p1, plan.p2, plan.base_exp
        B = 10 ** be
        inv = pow(p1, p2 - 2, p2)
        z1 = [int(halo[0]), int(halo[1])] + [int(v) for v in z[0].tolist()]
        z2 = [int(halo[2]), int(halo[3])] + [int(v) for v in z[1].tolist()]
        coef = [a1 + p1 * ((a2 - a1) * inv % p2) for a1, a2 in zip(z1, z2)]
        digs = [(c % B, c // B % B, c // (B * B)) for c in coef]
        L = plan.local_len
        K = L + (2 if q == plan.ranks - 1 else 0)
        s = []
        n = len(digs)
        for k in range(K):  # s_k = d0[k] + d1[k-1] + d2[k-2]; digs[k + 2] is local coefficient k
            i = k + 2
            s.append((digs[i][0] if i < n else 0) + (digs[i - 1][1] if i - 1 < n else 0) + digs[i - 2][2])
        return s, B

    def carry_begin(self, plan, q, z, halo, s_buf, maps):
        s, B = self._limbs(plan, q, z, halo)
        m = 0x24
        for v in s:
            lm = sum(((v + c) // B) << (2 * c) for c in range(3))
            m = map_compose(lm, m)
        self._carry[q] = (s, B)
        return m

    def _values(self, q, cin):
        s, B = self._carry[q]
        out, c = [], cin
        for v in s:
            t = v + c
            out.append(t % B)
            c = t // B
        return out

    def carry_probe(self, plan, q, cin, z, s_buf, maps):
        vals = self._values(q, cin)
        k0 = q * plan.local_len
        res = []
        for t in (0, 1):
            kg = plan.top_candidates[t]
            res.append(vals[kg - k0] if k0 <= kg < k0 + len(vals) else 2**64 - 1)
        return res

    def carry_emit(self, plan, q, cin, top, top_len, z, s_buf, maps, out):
        vals = self._values(q, cin)
        be, k0 = plan.base_exp, q * plan.local_len
        for j, v in enumerate(vals):
            kg = k0 + j
            if kg > top:
                break
            pos = 0 if kg == top else top_len + (top - 1 - kg) * be
            txt = str(v) if kg == top else str(v).zfill(be)
            out[pos:pos + len(txt)] = torch.tensor(list(txt.encode()), dtype=torch.uint8)


__all__ = ["EmuBackend", "map_apply"]
