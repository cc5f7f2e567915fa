"""TEST INFRASTRUCTURE (oracle) — not product code.

ctypes front ends for the two CPU checkers built by ``oracle/Makefile``:

* :func:`port` — ``_build/liboracle.so``, the plain-C restatement of the
  reference hot path (``decmul_oracle.c``; each function cites reference file:line).
* :func:`ref` — ``_ref/libdecmul_ref.so``, the reference's own sources compiled
  unmodified (plus the extern "C" wrapper ``ref_capi.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
P1 = 9223372036015915009
P2 = 9223372036166909953

_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _build(target: str) -> None:
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


class _Lib:
    """Shared call helpers for both libraries (same argument conventions)."""

    prefix = ""

    def __init__(self, path: str):
        self.lib = C.CDLL(path)
        self.path = path

    def fn(self, name, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        return f

    def check(self, rc: int) -> None:
        if rc:
            err = self.fn("last_error", C.c_char_p)()
            raise OracleError(rc, err.decode() if err else f"rc={rc}")

    # ---- field ----
    def make_ctx(self, p: int):
        pp, r, r2 = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.check(self.fn("make_ctx")(C.c_uint64(p), C.byref(pp), C.byref(r), C.byref(r2)))
        return pp.value, r.value, r2.value

    def redc(self, p, x, y):
        return self.fn("redc", C.c_uint64)(C.c_uint64(p), C.c_uint64(x), C.c_uint64(y))

    def to_mont(self, p, x):
        return self.fn("to_mont", C.c_uint64)(C.c_uint64(p), C.c_uint64(x))

    def from_mont(self, p, x):
        return self.fn("from_mont", C.c_uint64)(C.c_uint64(p), C.c_uint64(x))

    def is_prime(self, n):
        return bool(self.fn("is_prime")(C.c_uint64(n)))

    def find_primes(self, w, n_min, ell):
        out = np.zeros(ell, np.uint64)
        self.check(self.fn("find_primes")(C.c_uint(w), C.c_uint(n_min), C.c_uint(ell), _ptr(out)))
        return [int(v) for v in out]

    def primitive_root(self, p, n):
        r = C.c_uint64()
        self.check(self.fn("primitive_root")(C.c_uint64(p), C.c_uint64(n), C.byref(r)))
        return r.value

    # ---- kernels ----
    def ntt_plan(self, p, n):
        fwd = np.zeros(max(n - 1, 1), np.uint64)
        inv = np.zeros(max(n - 1, 1), np.uint64)
        root, psi, psip = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.check(self.fn("ntt_plan")(C.c_uint64(p), C.c_size_t(n), _ptr(fwd), _ptr(inv), C.byref(root),
                                       C.byref(psi), C.byref(psip)))
        return dict(fwd=fwd[: n - 1], inv=inv[: n - 1], root=root.value, psi=psi.value, psi_prime=psip.value)

    def dif_forward(self, p, a):
        a = _u64(a).copy()
        self.check(self.fn("dif_forward")(C.c_uint64(p), C.c_size_t(a.size), _ptr(a)))
        return a

    def dit_inverse(self, p, a):
        a = _u64(a).copy()
        self.check(self.fn("dit_inverse")(C.c_uint64(p), C.c_size_t(a.size), _ptr(a)))
        return a

    def bit_rev_permute(self, a):
        a = _u64(a).copy()
        self.fn("bit_rev_permute", None)(_ptr(a), C.c_size_t(a.size))
        return a

    def transpose_square_sub(self, a, n, stride):
        a = _u64(a).copy()
        self.fn("transpose_square_sub", None)(_ptr(a), C.c_size_t(n), C.c_size_t(stride))
        return a

    def transpose_n_x_2n(self, a, n):
        a = _u64(a).copy()
        self.fn("transpose_n_x_2n", None)(_ptr(a), C.c_size_t(n))
        return a

    def transpose_2n_x_n(self, a, n):
        a = _u64(a).copy()
        self.fn("transpose_2n_x_n", None)(_ptr(a), C.c_size_t(n))
        return a

    # ---- convolution ----
    def forward_transform(self, p, a, thr=0):
        a = _u64(a).copy()
        self.check(self.fn("forward_transform")(C.c_uint64(p), C.c_size_t(a.size), C.c_size_t(thr), _ptr(a)))
        return a

    def inverse_transform(self, p, a, thr=0):
        a = _u64(a).copy()
        self.check(self.fn("inverse_transform")(C.c_uint64(p), C.c_size_t(a.size), C.c_size_t(thr), _ptr(a)))
        return a

    def pointwise_product(self, p, a, b):
        a = _u64(a).copy()
        b = a if b is None else _u64(b)
        self.check(self.fn("pointwise_product")(C.c_uint64(p), C.c_size_t(a.size), _ptr(a), _ptr(b)))
        return a

    def convolve_mod_p(self, p, n, x, y, thr=0):
        """y is None -> aliased squaring path (conv.cpp:299-300)."""
        x = _u64(x)
        yy = x if y is None else _u64(y)
        out = np.zeros(n, np.uint64)
        self.check(self.fn("convolve_mod_p")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(thr), _ptr(x),
                                             C.c_size_t(x.size), _ptr(yy), C.c_size_t(yy.size), _ptr(out)))
        return out

    # ---- decimal ----
    def pack(self, digits: bytes, base_exp: int):
        cap = len(digits) // max(base_exp, 1) + 2
        out = np.zeros(cap, np.uint64)
        nl = C.c_size_t()
        self.check(self.fn("pack")(digits, C.c_size_t(len(digits)), C.c_uint(base_exp), _ptr(out),
                                   C.c_size_t(cap), C.byref(nl)))
        return out[: nl.value].copy()

    def to_decimal(self, limbs, base_exp: int) -> bytes:
        limbs = _u64(limbs)
        cap = limbs.size * 20 + 2
        buf = C.create_string_buffer(cap)
        ln = C.c_size_t()
        self.check(self.fn("to_decimal")(_ptr(limbs), C.c_size_t(limbs.size), C.c_uint(base_exp), buf,
                                         C.c_size_t(cap), C.byref(ln)))
        return buf.raw[: ln.value]

    def crt2(self, p1, p2, a1, a2) -> int:
        lo, hi = C.c_uint64(), C.c_uint64()
        self.check(self.fn("crt2")(C.c_uint64(p1), C.c_uint64(p2), C.c_uint64(a1), C.c_uint64(a2), C.byref(lo),
                                   C.byref(hi)))
        return (hi.value << 64) | lo.value

    def recover_digits(self, coeffs, base_exp, min_limbs):
        """coeffs: iterable of python ints < 2^128 or an (n,2) uint64 array (lo, hi)."""
        arr = np.asarray(coeffs)
        if arr.dtype != np.uint64 or arr.ndim != 2:
            arr = np.array([[int(c) & (2**64 - 1), int(c) >> 64] for c in coeffs], dtype=np.uint64).reshape(-1, 2)
        arr = np.ascontiguousarray(arr)
        n = arr.shape[0]
        cap = n + 4
        out = np.zeros(cap, np.uint64)
        nout = C.c_size_t()
        self.check(self.fn("recover_digits")(_ptr(arr), C.c_size_t(n), C.c_uint(base_exp), C.c_size_t(min_limbs),
                                             _ptr(out), C.c_size_t(cap), C.byref(nout)))
        return out[: nout.value].copy()


class Port(_Lib):
    prefix = "or_"

    def conv_plan_info(self, p, n, thr=0):
        shape, root, psi, psip = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        n1, n2 = C.c_size_t(), C.c_size_t()
        self.check(self.fn("conv_plan_info")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(thr), C.byref(shape),
                                             C.byref(root), C.byref(psi), C.byref(psip), C.byref(n1), C.byref(n2)))
        return dict(shape=shape.value, root=root.value, psi=psi.value, psi_prime=psip.value, n1=n1.value, n2=n2.value)

    def smallest_supported_length(self, need, p1=0, p2=0):
        out = C.c_size_t()
        self.check(self.fn("smallest_supported_length")(C.c_size_t(need), C.c_uint64(p1), C.c_uint64(p2),
                                                        C.byref(out)))
        return out.value

    def select_base_and_length(self, dx, dy, forced=0, p1=0, p2=0):
        be, ln = C.c_uint(), C.c_size_t()
        self.check(self.fn("select_base_and_length")(C.c_size_t(dx), C.c_size_t(dy), C.c_uint64(p1),
                                                     C.c_uint64(p2), C.c_uint(forced), C.byref(be), C.byref(ln)))
        return be.value, ln.value

    def multiply(self, x: bytes, y: bytes | None = None, forced=0, p1=0, p2=0) -> bytes:
        y = x if y is None else y
        cap = len(x) + len(y) + 2
        buf = C.create_string_buffer(cap)
        ln = C.c_size_t()
        self.check(self.fn("multiply")(x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), buf, C.c_size_t(cap),
                                       C.byref(ln), C.c_uint(forced), C.c_uint64(p1), C.c_uint64(p2)))
        return buf.raw[: ln.value]

    def naive_dft(self, x, root, p):
        x = _u64(x)
        out = np.zeros(x.size, np.uint64)
        self.check(self.fn("naive_dft")(_ptr(x), C.c_size_t(x.size), C.c_uint64(root), C.c_uint64(p), _ptr(out)))
        return out

    def naive_convolve(self, x, y, p):
        x, y = _u64(x), _u64(y)
        out = np.zeros(x.size, np.uint64)
        self.check(self.fn("naive_convolve")(_ptr(x), _ptr(y), C.c_size_t(x.size), C.c_uint64(p), _ptr(out)))
        return out

    def schoolbook_multiply(self, x: bytes, y: bytes) -> bytes:
        cap = len(x) + len(y) + 2
        buf = C.create_string_buffer(cap)
        ln = C.c_size_t()
        self.check(self.fn("schoolbook_multiply")(x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), buf,
                                                  C.c_size_t(cap), C.byref(ln)))
        return buf.raw[: ln.value]

    def gen_digits(self, seed: int, n: int, mode: int = 0) -> bytes:
        buf = C.create_string_buffer(n)
        self.fn("gen_digits", None)(C.c_uint64(seed), C.c_int(mode), C.c_size_t(n), buf)
        return buf.raw[:n]

    def dif_forward_root(self, p, a, root):
        a = _u64(a).copy()
        self.check(self.fn("dif_forward_root")(C.c_uint64(p), C.c_size_t(a.size), C.c_uint64(root), _ptr(a)))
        return a

    def ntt_plan_root(self, p, n, root):
        fwd = np.zeros(max(n - 1, 1), np.uint64)
        inv = np.zeros(max(n - 1, 1), np.uint64)
        self.check(self.fn("ntt_plan_root")(C.c_uint64(p), C.c_size_t(n), C.c_uint64(root), _ptr(fwd), _ptr(inv)))
        return fwd[: n - 1], inv[: n - 1]

    def residue_mod(self, s: bytes, q: int) -> int:
        return self.fn("residue_mod", C.c_uint64)(s, C.c_size_t(len(s)), C.c_uint64(q))

    def residues(self, digits, qs, threads: int = 0) -> list[int]:
        """Residues of a digit string (bytes or uint8 ndarray) modulo each q in qs; the
        string is cut into per-thread slices (the C call releases the GIL) and the slice
        residues are combined as r(ab) = r(a) 10^|b| + r(b)."""
        from concurrent.futures import ThreadPoolExecutor

        a = np.frombuffer(digits, dtype=np.uint8) if isinstance(digits, (bytes, bytearray)) else digits
        n, nq = a.size, len(qs)
        threads = threads or (os.cpu_count() or 1)
        cuts = [n * t // threads for t in range(threads + 1)]
        qarr = np.array(qs, dtype=np.uint64)
        fn = self.fn("residues_multi", None)

        def one(t):
            out = np.zeros(nq, np.uint64)
            lo, hi = cuts[t], cuts[t + 1]
            fn(C.c_void_p(a.ctypes.data + lo), C.c_size_t(hi - lo), _ptr(qarr), C.c_int(nq), _ptr(out))
            return [int(v) for v in out], hi - lo

        with ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(one, range(threads)))
        res = [0] * nq
        for r, ln in parts:
            res = [(res[k] * pow(10, ln, qs[k]) + r[k]) % qs[k] for k in range(nq)]
        return res

    def add_shifted(self, acc: np.ndarray, p: bytes, shift: int) -> None:
        """acc (little-endian uint8 decimal digits) += int(p) * 10^shift, exactly."""
        rc = self.fn("add_shifted")(C.c_void_p(acc.ctypes.data), C.c_size_t(acc.size), p, C.c_size_t(len(p)),
                                    C.c_size_t(shift))
        if rc:
            raise OracleError(rc, "add_shifted: sum does not fit the accumulator")

    def carry_u16(self, acc: np.ndarray) -> bytes:
        """Decimal string (most significant first, leading zeros stripped) of a carry-free
        little-endian uint16 digit-column accumulator."""
        out = C.create_string_buffer(acc.size + 1)
        rc = self.fn("carry_u16")(C.c_void_p(acc.ctypes.data), C.c_size_t(acc.size), out)
        if rc:
            raise OracleError(rc, "carry_u16: carry overflow")
        return out.raw[: acc.size + 1].lstrip(b"0") or b"0"

    def gen_residues(self, seed: int, n: int, p: int):
        out = np.zeros(n, np.uint64)
        self.fn("gen_residues", None)(C.c_uint64(seed), C.c_size_t(n), C.c_uint64(p), _ptr(out))
        return out


class Ref(_Lib):
    prefix = "ref_"

    def conv_plan_info(self, p, n, thr=0):
        shape, root, psi, psip = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        n1, n2, cr, rr = C.c_size_t(), C.c_size_t(), C.c_uint64(), C.c_uint64()
        self.check(self.fn("conv_plan_info")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(thr), C.byref(shape),
                                             C.byref(root), C.byref(psi), C.byref(psip), C.byref(n1), C.byref(n2),
                                             C.byref(cr), C.byref(rr)))
        return dict(shape=shape.value, root=root.value, psi=psi.value, psi_prime=psip.value, n1=n1.value,
                    n2=n2.value, col_root=cr.value, row_root=rr.value)

    def smallest_supported_length(self, need, p1=0, p2=0):
        out = C.c_size_t()
        if p1:
            self.check(self.fn("smallest_supported_length_pair")(C.c_size_t(need), C.c_uint64(p1), C.c_uint64(p2),
                                                                 C.byref(out)))
        else:
            self.check(self.fn("smallest_supported_length")(C.c_size_t(need), C.byref(out)))
        return out.value

    def select_base_and_length(self, dx, dy, forced=0, p1=0, p2=0):
        be, ln = C.c_uint(), C.c_size_t()
        if p1:
            self.check(self.fn("select_base_and_length_pair")(C.c_size_t(dx), C.c_size_t(dy), C.c_uint64(p1),
                                                              C.c_uint64(p2), C.c_uint(forced), C.byref(be),
                                                              C.byref(ln)))
        else:
            self.check(self.fn("select_base_and_length")(C.c_size_t(dx), C.c_size_t(dy), C.c_uint(forced),
                                                         C.byref(be), C.byref(ln)))
        return be.value, ln.value

    def multiply(self, x: bytes, y: bytes | None = None, forced=0, strategy=1) -> bytes:
        alias = y is None
        y = x if y is None else y
        cap = len(x) + len(y) + 2
        buf = C.create_string_buffer(cap)
        ln = C.c_size_t()
        self.check(self.fn("multiply")(x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), buf, C.c_size_t(cap),
                                       C.byref(ln), C.c_uint(forced), C.c_int(strategy), C.c_int(int(alias))))
        return buf.raw[: ln.value]

    def multiply_batch(self, xs: list[bytes], ys: list[bytes], threads: int) -> list[bytes]:
        n = len(xs)
        xo = np.cumsum([0] + [len(v) for v in xs[:-1]]).astype(np.uintp)
        yo = np.cumsum([0] + [len(v) for v in ys[:-1]]).astype(np.uintp)
        nx = np.array([len(v) for v in xs], np.uintp)
        ny = np.array([len(v) for v in ys], np.uintp)
        cap = nx + ny + 1
        oo = np.cumsum(np.concatenate([[0], cap[:-1]])).astype(np.uintp)
        outs = C.create_string_buffer(int(cap.sum()))
        olen = np.zeros(n, np.uintp)
        szp = lambda a: a.ctypes.data_as(_szp)  # noqa: E731
        self.check(self.fn("multiply_batch")(C.c_size_t(n), b"".join(xs), szp(xo), szp(nx), b"".join(ys), szp(yo),
                                             szp(ny), outs, szp(oo), szp(cap), szp(olen), C.c_int(threads)))
        raw = outs.raw
        return [raw[int(oo[i]): int(oo[i]) + int(olen[i])] for i in range(n)]

    def bench_inputs(self, digits: int, seed: int = 42):
        x = C.create_string_buffer(digits)
        y = C.create_string_buffer(digits)
        self.fn("bench_inputs", None)(C.c_size_t(digits), C.c_uint64(seed), x, y)
        return x.raw[:digits], y.raw[:digits]

    def random_residues(self, seed, n, p):
        out = np.zeros(n, np.uint64)
        self.fn("random_residues", None)(C.c_uint64(seed), C.c_size_t(n), C.c_uint64(p), _ptr(out))
        return out


_port = None
_ref = None


def port() -> Port:
    """The plain-C restatement (built on demand with gcc)."""
    global _port
    if _port is None:
        path = os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(os.path.join(HERE, "decmul_oracle.c")):
            _build("oracle")
        _port = Port(path)
    return _port


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libdecmul_ref.so")) or os.path.isdir("/root/reference/proj/src")


def ref() -> Ref:
    """The reference's own sources compiled unmodified (built here; prebuilt .so on the GPU box)."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libdecmul_ref.so")
        if not os.path.exists(path):
            _build("ref")
        _ref = Ref(path)
    return _ref
