"""B200-native decimal multiplier — Python mirror of the reference ``decmul`` API.

The product is ``libdecmul_gpu.so`` (hand-written sm_100a kernels behind the C ABI
``include/decmul_gpu.h``). This module binds that C ABI with ctypes and re-exposes
the reference's C++ API names (``proj/include/decmul/decimal.hpp``,
``conv.hpp``, ``transpose.hpp``) with the same argument meaning and error types:

* ``DecimalNumber.parse`` / ``multiply`` / ``MultiplyOptions`` / ``OperandTooLarge``
  (decimal.hpp:20-38, :170-177)
* ``select_base_and_length`` / ``smallest_supported_length`` (decimal.hpp:66-76)
* ``pack`` / ``to_decimal`` (decimal.hpp:78-82)
* ``convolve_mod_p`` / ``forward_transform`` / ``inverse_transform`` /
  ``pointwise_product`` (conv.hpp:59-71)
* ``transpose_square_sub`` / ``transpose_n_x_2n`` / ``transpose_2n_x_n``
  (transpose.hpp:11-24)

There is no CPU fallback: if the CUDA library is missing or no GPU is visible,
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "P1", "P2", "Q1", "Q2", "OperandTooLarge", "CudaError", "DecimalNumber", "MultiplyOptions", "BasePlan",
    "PackedOperand", "Context", "default_context", "multiply", "multiply_batch", "select_base_and_length",
    "smallest_supported_length", "pack", "to_decimal", "convolve_mod_p", "forward_transform",
    "inverse_transform", "build_conv_plan", "pointwise_product", "transpose_square_sub", "transpose_n_x_2n", "transpose_2n_x_n",
    "lib_path", "load_library", "EXPORTED_SYMBOLS",
]

P1 = 9223372036015915009  # reference primes.hpp:30
P2 = 9223372036166909953  # reference primes.hpp:31
Q1 = 9223371938070528001  # find_primes(64, 30, 2) (primes.cpp:70-81): lengths beyond 3 * 2^24
Q2 = 9223371941291753473

HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    """The in-tree library; DECMUL_GPU_LIB overrides the path (A/B timing of kernel variants)."""
    return os.environ.get("DECMUL_GPU_LIB") or os.path.join(HERE, "libdecmul_gpu.so")


# every function declared in include/decmul_gpu.h
EXPORTED_SYMBOLS = [
    "decmul_gpu_create", "decmul_gpu_destroy", "decmul_gpu_last_error", "decmul_gpu_device_count",
    "decmul_gpu_select_base_and_length", "decmul_gpu_smallest_supported_length", "decmul_gpu_plan",
    "decmul_gpu_multiply", "decmul_gpu_multiply_device", "decmul_gpu_result_length", "decmul_gpu_multiply_batch",
    "decmul_gpu_multiply_batch_device", "decmul_gpu_convolve_mod_p", "decmul_gpu_forward_transform",
    "decmul_gpu_inverse_transform", "decmul_gpu_pointwise_product", "decmul_gpu_pack",
    "decmul_gpu_recover_decimal", "decmul_gpu_transpose_square_sub", "decmul_gpu_transpose_n_x_2n",
    "decmul_gpu_transpose_2n_x_n", "decmul_gpu_generate_digits", "decmul_gpu_measure_modmul_rate",
    "decmul_gpu_get_stats", "decmul_gpu_shard_plan_create", "decmul_gpu_shard_pack", "decmul_gpu_shard_transform",
    "decmul_gpu_shard_reorder", "decmul_gpu_shard_carry_begin", "decmul_gpu_shard_carry_probe",
    "decmul_gpu_shard_carry_emit", "decmul_gpu_selftest", "decmul_gpu_multiply_batch_ptrs",
    "decmul_gpu_check_errors", "decmul_gpu_profile", "decmul_gpu_profile_report", "decmul_gpu_create_multi",
    "decmul_gpu_context_devices", "decmul_gpu_multiply_sharded", "decmul_gpu_multiply_ex",
    "decmul_gpu_coalesce_stats", "decmul_gpu_forward_transform_ex", "decmul_gpu_inverse_transform_ex",
    "decmul_gpu_conv_plan_info",
]


class OperandTooLarge(RuntimeError):
    """decmul::OperandTooLarge (reference decimal.hpp:20-22)."""


class CudaError(RuntimeError):
    pass


class LogicError(RuntimeError):
    """std::logic_error from an internal self-check."""


_ERRORS = {1: ValueError, 2: OperandTooLarge, 3: RuntimeError, 4: LogicError, 5: CudaError, 6: MemoryError,
           7: BufferError}

_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


class _PlanInfo(C.Structure):
    _fields_ = [("base_exp", C.c_uint), ("length", C.c_size_t), ("p1", C.c_uint64), ("p2", C.c_uint64),
                ("large_pair", C.c_int), ("one_cta", C.c_int)]


class _MulOpts(C.Structure):
    _fields_ = [("forced_base_exp", C.c_uint), ("p1", C.c_uint64), ("p2", C.c_uint64), ("alias", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("last_launches", C.c_int), ("table_bytes", C.c_size_t)]


_lib = None


def load_library():
    """Load libdecmul_gpu.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = C.CDLL(path)
        lib.decmul_gpu_last_error.restype = C.c_char_p
        lib.decmul_gpu_last_error.argtypes = [C.c_void_p]
        lib.decmul_gpu_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
        lib.decmul_gpu_destroy.argtypes = [C.c_void_p]
        lib.decmul_gpu_destroy.restype = None
        _lib = lib
    return _lib


def _raise(rc: int, ctx) -> None:
    if rc == 0:
        return
    msg = load_library().decmul_gpu_last_error(ctx)
    msg = msg.decode() if msg else f"decmul_gpu error {rc}"
    raise _ERRORS.get(rc, RuntimeError)(msg)


def _u64arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


@dataclass
class BasePlan:
    """reference decimal.hpp:61-64"""
    base_exp: int
    length: int


@dataclass
class PackedOperand:
    """reference decimal.hpp:41-44"""
    base_exp: int
    limbs: np.ndarray


@dataclass
class MultiplyOptions:
    """reference decimal.hpp:170-173. ``strategy`` is the reference's CPU codegen
    knob (words.hpp:29); products are identical under both, so it is accepted
    and ignored. ``primes`` (extension): the planner's prime pair (p1, p2), which the
    reference's multiply pins to production_primes() (decimal.cpp:194); None = the
    reference pair, or the large pair beyond its 3 * 2^24 cap."""
    strategy: int = 1
    forced_base_exp: int = 0
    primes: tuple[int, int] | None = None


class DecimalNumber:
    """Non-negative integer as canonical ASCII digits (reference decimal.hpp:26-38)."""

    __slots__ = ("_text",)

    def __init__(self, text: bytes = b"0", _trusted: bool = False):
        if not _trusted:
            text = DecimalNumber.parse(text)._text
        self._text = bytes(text)

    @staticmethod
    def parse(text) -> "DecimalNumber":
        """reference decimal.cpp:29-36 (same messages)."""
        if isinstance(text, str):
            text = text.encode()
        text = bytes(text)
        if not text:
            raise ValueError("decimal: empty string")
        arr = np.frombuffer(text, dtype=np.uint8)
        if ((arr < 48) | (arr > 57)).any():
            raise ValueError("decimal: non-digit character")
        if len(text) > 1 and text[:1] == b"0":
            raise ValueError("decimal: leading zero")
        return DecimalNumber(text, _trusted=True)

    def text(self) -> bytes:
        return self._text

    def digit_count(self) -> int:
        return len(self._text)

    def is_zero(self) -> bool:
        return self._text == b"0"

    def __eq__(self, other):
        return isinstance(other, DecimalNumber) and other._text == self._text

    def __repr__(self):
        t = self._text
        return f"DecimalNumber({t[:20].decode()}{'...' if len(t) > 20 else ''}, digits={len(t)})"


class Context:
    """A device context (``decmul_gpu_ctx``): plan cache, workspace, streams. ``devices`` (a
    list) makes a multi-GPU context (decmul_gpu_create_multi): host-buffer products fan out
    over the devices and large single products are sharded; device ids may repeat."""

    def __init__(self, device: int = 0, devices: list[int] | None = None):
        lib = load_library()
        h = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*devices)
            rc = lib.decmul_gpu_create_multi(C.byref(h), arr, C.c_int(len(devices)))
            device = devices[0]
        else:
            rc = lib.decmul_gpu_create(C.byref(h), C.c_int(device))
        if rc:
            _raise(rc, None)
        self._h = h
        self._lib = lib
        self.device = device

    def devices(self) -> list[int]:
        arr = (C.c_int * 64)()
        n = C.c_int()
        self._call("decmul_gpu_context_devices", arr, C.c_int(64), C.byref(n))
        return list(arr[: n.value])

    def multiply_sharded(self, x: bytes, y: bytes | None) -> bytes:
        """The product sharded over the context's devices whatever its size (parity tests)."""
        alias = y is None
        y = x if alias else y
        cap = len(x) + len(y) + 1
        out = C.create_string_buffer(cap)
        n = C.c_size_t()
        self._call("decmul_gpu_multiply_sharded", x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), out,
                   C.c_size_t(cap), C.byref(n), C.c_int(int(alias)))
        return out.raw[: n.value]

    def close(self):
        if getattr(self, "_h", None):
            self._lib.decmul_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, name, *args):
        rc = getattr(self._lib, name)(self._h, *args)
        _raise(rc, self._h)

    # ---- planning ----
    def plan(self, dx: int, dy: int, forced_base_exp: int = 0) -> dict:
        info = _PlanInfo()
        self._call("decmul_gpu_plan", C.c_size_t(dx), C.c_size_t(dy), C.c_uint(forced_base_exp), C.byref(info))
        return dict(base_exp=info.base_exp, length=info.length, p1=info.p1, p2=info.p2,
                    large_pair=bool(info.large_pair), one_cta=bool(info.one_cta))

    def selftest(self, inject_fault: bool = False) -> tuple[int, str]:
        """GPU self-test (reference run_selftest, selftest.cpp:79-219): (failures, report)."""
        buf = C.create_string_buffer(1 << 14)
        f = C.c_int()
        self._call("decmul_gpu_selftest", C.c_int(int(inject_fault)), buf, C.c_size_t(len(buf)), C.byref(f))
        return f.value, buf.value.decode()

    def stats(self) -> dict:
        s = _Stats()
        self._call("decmul_gpu_get_stats", C.byref(s))
        return dict(last_launches=s.last_launches, table_bytes=s.table_bytes)

    def coalesce_stats(self) -> tuple[int, int]:
        """(batches, products) run by the coalescing path of concurrent small multiplies."""
        b, p = C.c_ulonglong(), C.c_ulonglong()
        self._call("decmul_gpu_coalesce_stats", C.byref(b), C.byref(p))
        return b.value, p.value

    def check_errors(self, stream: int = 0) -> None:
        """Raise the errors of the asynchronous entry points since the last check (syncs stream)."""
        self._call("decmul_gpu_check_errors", C.c_void_p(stream))

    def profile(self, enable: bool = True) -> None:
        """Per-launch CUDA-event timing of every kernel this context enqueues."""
        self._call("decmul_gpu_profile", C.c_int(int(enable)))

    def profile_report(self) -> list[tuple[str, float, float, float]]:
        """[(kernel name, ms, algorithmic modmuls, algorithmic HBM bytes)] since the last report."""
        n = C.c_size_t()
        self._call("decmul_gpu_profile_report", None, C.c_size_t(0), C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        self._call("decmul_gpu_profile_report", buf, C.c_size_t(len(buf)), C.byref(n))
        out = []
        for line in buf.value.decode().splitlines():
            name, ms, mm, by = line.split("\t")
            out.append((name, float(ms), float(mm), float(by)))
        return out

    # ---- multiply ----
    def multiply_text(self, x: bytes, y: bytes | None, forced_base_exp: int = 0,
                      primes: tuple[int, int] | None = None) -> bytes:
        """Digits in host memory -> product digits. y=None is the aliased squaring path;
        primes = the planner's prime pair (decmul_gpu_multiply_ex), None = automatic."""
        alias = y is None
        y = x if alias else y
        cap = len(x) + len(y) + 1
        out = C.create_string_buffer(cap)
        n = C.c_size_t()
        if primes is None:
            self._call("decmul_gpu_multiply", x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), out, C.c_size_t(cap),
                       C.byref(n), C.c_uint(forced_base_exp), C.c_int(int(alias)))
        else:
            o = _MulOpts(forced_base_exp, primes[0], primes[1], int(alias))
            self._call("decmul_gpu_multiply_ex", x, C.c_size_t(len(x)), y, C.c_size_t(len(y)), out,
                       C.c_size_t(cap), C.byref(n), C.byref(o))
        return out.raw[: n.value]

    def multiply_ptr(self, h_x: int, nx: int, h_y: int, ny: int, h_out: int, cap: int, alias: bool = False,
                     forced_base_exp: int = 0) -> int:
        """Host pointers (ints, e.g. pinned torch tensor.data_ptr()); returns the product length.
        Thread-safe; concurrent calls with large pinned buffers overlap their transfers
        (one call's download with the next call's upload and compute)."""
        n = C.c_size_t()
        self._call("decmul_gpu_multiply", C.c_void_p(h_x), C.c_size_t(nx), C.c_void_p(h_y), C.c_size_t(ny),
                   C.c_void_p(h_out), C.c_size_t(cap), C.byref(n), C.c_uint(forced_base_exp), C.c_int(int(alias)))
        return n.value

    def multiply_device(self, d_x: int, nx: int, d_y: int, ny: int, d_out: int, cap: int, stream: int = 0,
                        squaring: bool = False, sync: bool = True, forced_base_exp: int = 0):
        """Device pointers (ints, e.g. torch tensor.data_ptr()); returns the length if sync."""
        n = C.c_size_t()
        self._call("decmul_gpu_multiply_device", C.c_void_p(d_x), C.c_size_t(nx), C.c_void_p(d_y),
                   C.c_size_t(ny), C.c_void_p(d_out), C.c_size_t(cap), C.byref(n) if sync else None,
                   C.c_uint(forced_base_exp), C.c_int(int(squaring)), C.c_void_p(stream))
        return n.value if sync else None

    def result_length(self) -> int:
        n = C.c_size_t()
        self._call("decmul_gpu_result_length", C.byref(n))
        return n.value

    def multiply_batch(self, xs: bytes, ys: bytes, count: int, nx: int, ny: int) -> list[bytes]:
        """Uniform-size batch from packed host buffers (operand i at i*nx / i*ny)."""
        stride = nx + ny
        outs = C.create_string_buffer(count * stride)
        lens = (C.c_size_t * count)()
        self._call("decmul_gpu_multiply_batch", C.c_size_t(count), xs, C.c_size_t(nx), C.c_size_t(nx), ys,
                   C.c_size_t(ny), C.c_size_t(ny), outs, C.c_size_t(stride), lens)
        raw = outs.raw
        return [raw[i * stride: i * stride + lens[i]] for i in range(count)]

    def multiply_batch_device(self, count, d_xs, nx, d_ys, ny, d_outs, out_stride, d_lens, stream=0,
                              x_stride=None, y_stride=None):
        self._call("decmul_gpu_multiply_batch_device", C.c_size_t(count), C.c_void_p(d_xs),
                   C.c_size_t(nx if x_stride is None else x_stride), C.c_size_t(nx), C.c_void_p(d_ys),
                   C.c_size_t(ny if y_stride is None else y_stride), C.c_size_t(ny), C.c_void_p(d_outs),
                   C.c_size_t(out_stride), C.c_void_p(d_lens), C.c_void_p(stream))

    def multiply_batch_mixed(self, xs: list, ys: list) -> list:
        """Products of mixed sizes (decmul_gpu_multiply_batch_ptrs): equal size pairs batched."""
        n = len(xs)
        if len(ys) != n:
            raise ValueError("multiply_batch_mixed: xs and ys differ in length")
        xb = [bytes(x) for x in xs]
        yb = [bytes(y) for y in ys]
        outs = [C.create_string_buffer(len(a) + len(b) + 1) for a, b in zip(xb, yb)]
        arr = lambda T, v: (T * n)(*v)  # noqa: E731
        lens = (C.c_size_t * n)()
        self._call("decmul_gpu_multiply_batch_ptrs", C.c_size_t(n), arr(C.c_char_p, xb),
                   arr(C.c_size_t, [len(a) for a in xb]), arr(C.c_char_p, yb), arr(C.c_size_t, [len(b) for b in yb]),
                   arr(C.c_void_p, [C.addressof(o) for o in outs]), arr(C.c_size_t, [len(o) for o in outs]), lens)
        return [o.raw[: lens[i]] for i, o in enumerate(outs)]

    def multiply_batch_ptr(self, count: int, xs_ptr: int, nx: int, ys_ptr: int, ny: int, outs_ptr: int,
                           out_stride: int, lens_ptr: int) -> None:
        """Uniform-size batch from caller-owned HOST buffers given as raw pointers (pinned
        memory from torch, say); lens_ptr receives size_t lengths."""
        self._call("decmul_gpu_multiply_batch", C.c_size_t(count), C.c_void_p(xs_ptr), C.c_size_t(nx),
                   C.c_size_t(nx), C.c_void_p(ys_ptr), C.c_size_t(ny), C.c_size_t(ny), C.c_void_p(outs_ptr),
                   C.c_size_t(out_stride), C.c_void_p(lens_ptr))

    def generate_digits(self, d_out: int, n: int, seed0: int, count: int = 1, seed_step: int = 1,
                        stride: int | None = None, mode: int = 0, stream: int = 0) -> None:
        """Seeded digits written in place on the device (same stream as inputs.gen_digits)."""
        self._call("decmul_gpu_generate_digits", C.c_uint64(seed0), C.c_uint64(seed_step), C.c_size_t(count),
                   C.c_size_t(n), C.c_size_t(n if stride is None else stride), C.c_int(mode), C.c_void_p(d_out),
                   C.c_void_p(stream))

    def measure_modmul_rate(self, variant: int = 0) -> float:
        r = C.c_double()
        self._call("decmul_gpu_measure_modmul_rate", C.c_int(variant), C.byref(r))
        return r.value

    # ---- parity hooks ----
    def convolve_mod_p(self, p: int, n: int, x, y=None) -> np.ndarray:
        x = _u64arr(x)
        yy = x if y is None else _u64arr(y)
        out = np.zeros(max(n, 1), np.uint64)
        self._call("decmul_gpu_convolve_mod_p", C.c_uint64(p), C.c_size_t(n), _ptr(x), C.c_size_t(x.size),
                   _ptr(yy), C.c_size_t(yy.size), _ptr(out))
        return out[:n]

    def forward_transform(self, p: int, a, six_step_threshold: int = 0) -> np.ndarray:
        """Spectrum in the storage order of build_conv_plan(ctx, n, six_step_threshold)
        (reference conv.hpp:19-24, :59-60; 0 = the default 2^15)."""
        a = _u64arr(a).copy()
        self._call("decmul_gpu_forward_transform_ex", C.c_uint64(p), C.c_size_t(a.size),
                   C.c_size_t(six_step_threshold), _ptr(a))
        return a

    def inverse_transform(self, p: int, a, six_step_threshold: int = 0) -> np.ndarray:
        a = _u64arr(a).copy()
        self._call("decmul_gpu_inverse_transform_ex", C.c_uint64(p), C.c_size_t(a.size),
                   C.c_size_t(six_step_threshold), _ptr(a))
        return a

    def pointwise_product(self, p: int, a, b=None) -> np.ndarray:
        a = _u64arr(a).copy()
        b = a.copy() if b is None else _u64arr(b)
        self._call("decmul_gpu_pointwise_product", C.c_uint64(p), C.c_size_t(a.size), _ptr(a), _ptr(b))
        return a

    def pack(self, digits: bytes, base_exp: int) -> np.ndarray:
        cap = len(digits) // max(base_exp, 1) + 2
        out = np.zeros(cap, np.uint64)
        n = C.c_size_t()
        self._call("decmul_gpu_pack", digits, C.c_size_t(len(digits)), C.c_uint(base_exp), _ptr(out),
                   C.c_size_t(cap), C.byref(n))
        return out[: n.value].copy()

    def recover_decimal(self, r1, r2, p1: int, p2: int, base_exp: int, min_limbs: int, digits_sum: int) -> bytes:
        r1, r2 = _u64arr(r1), _u64arr(r2)
        cap = max(digits_sum, 1) + 64
        out = C.create_string_buffer(cap)
        n = C.c_size_t()
        self._call("decmul_gpu_recover_decimal", _ptr(r1), _ptr(r2), C.c_size_t(r1.size), C.c_uint64(p1),
                   C.c_uint64(p2), C.c_uint(base_exp), C.c_size_t(min_limbs), C.c_size_t(digits_sum), out,
                   C.c_size_t(cap), C.byref(n))
        return out.raw[: n.value]

    def transpose_square_sub(self, a, n: int, stride: int) -> np.ndarray:
        a = _u64arr(a).copy()
        self._call("decmul_gpu_transpose_square_sub", _ptr(a), C.c_size_t(n), C.c_size_t(stride))
        return a

    def transpose_n_x_2n(self, a, n: int) -> np.ndarray:
        a = _u64arr(a).copy()
        self._call("decmul_gpu_transpose_n_x_2n", _ptr(a), C.c_size_t(n))
        return a

    def transpose_2n_x_n(self, a, n: int) -> np.ndarray:
        a = _u64arr(a).copy()
        self._call("decmul_gpu_transpose_2n_x_n", _ptr(a), C.c_size_t(n))
        return a


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default


# ---------------- reference-shaped free functions ----------------

def smallest_supported_length(need: int, pair: tuple[int, int] | None = None) -> int:
    """reference decimal.cpp:54-76; returns 0 when no supported length is large enough."""
    p1, p2 = pair if pair else (0, 0)
    out = C.c_size_t()
    _raise(load_library().decmul_gpu_smallest_supported_length(C.c_size_t(need), C.c_uint64(p1), C.c_uint64(p2),
                                                              C.byref(out)), None)
    return out.value


def select_base_and_length(dx: int, dy: int, pair: tuple[int, int] | None = None,
                           forced_base_exp: int = 0) -> BasePlan:
    """reference decimal.cpp:78-100 (raises OperandTooLarge / ValueError like the reference)."""
    p1, p2 = pair if pair else (0, 0)
    be, ln = C.c_uint(), C.c_size_t()
    _raise(load_library().decmul_gpu_select_base_and_length(C.c_size_t(dx), C.c_size_t(dy), C.c_uint64(p1),
                                                           C.c_uint64(p2), C.c_uint(forced_base_exp),
                                                           C.byref(be), C.byref(ln)), None)
    return BasePlan(be.value, ln.value)


def build_conv_plan(p: int, n: int, six_step_threshold: int = 0) -> dict:
    """reference build_conv_plan (conv.hpp:59-60, conv.cpp:212-271): shape ("direct", "six_step",
    "three_rows"), plain primitive root and six-step factors of the plan; needs no GPU. Raises
    ValueError like the reference's invalid_argument."""
    shape, root, n1, n2 = C.c_int(), C.c_uint64(), C.c_size_t(), C.c_size_t()
    _raise(load_library().decmul_gpu_conv_plan_info(C.c_uint64(p), C.c_size_t(n), C.c_size_t(six_step_threshold),
                                                   C.byref(shape), C.byref(root), C.byref(n1), C.byref(n2)), None)
    return dict(p=p, n=n, six_step_threshold=six_step_threshold or 1 << 15,
                shape=("direct", "six_step", "three_rows")[shape.value], root=root.value, n1=n1.value, n2=n2.value)


def multiply(x: DecimalNumber, y: DecimalNumber, opt: MultiplyOptions | None = None,
             ctx: Context | None = None) -> DecimalNumber:
    """reference decimal.cpp:191-216: exact product; x is y takes the squaring path."""
    opt = opt or MultiplyOptions()
    ctx = ctx or default_context()
    if x.is_zero() or y.is_zero():
        return DecimalNumber()
    z = ctx.multiply_text(x.text(), None if x is y else y.text(), opt.forced_base_exp, opt.primes)
    return DecimalNumber(z, _trusted=True)


def multiply_batch(xs: list[DecimalNumber], ys: list[DecimalNumber], ctx: Context | None = None):
    """Independent products of uniform sizes in one launch (falls back to per-product calls otherwise)."""
    ctx = ctx or default_context()
    if not xs:
        return []
    nx, ny = xs[0].digit_count(), ys[0].digit_count()
    if all(v.digit_count() == nx for v in xs) and all(v.digit_count() == ny for v in ys):
        outs = ctx.multiply_batch(b"".join(v.text() for v in xs), b"".join(v.text() for v in ys), len(xs), nx, ny)
        return [DecimalNumber(o, _trusted=True) for o in outs]
    return [multiply(a, b, ctx=ctx) for a, b in zip(xs, ys)]


def pack(x: DecimalNumber, base_exp: int, ctx: Context | None = None) -> PackedOperand:
    """reference decimal.cpp:102-118 (on the device)."""
    if base_exp < 1 or base_exp > 17:
        raise ValueError("pack: unsupported base")
    return PackedOperand(base_exp, (ctx or default_context()).pack(x.text(), base_exp))


def to_decimal(x: PackedOperand) -> bytes:
    """reference decimal.cpp:120-134 (host formatting of a limb vector; the device path formats
    inside the carry kernel)."""
    limbs = [int(v) for v in np.asarray(x.limbs, dtype=np.uint64)]
    top = len(limbs)
    while top > 1 and limbs[top - 1] == 0:
        top -= 1
    if top == 0:
        return b"0"
    parts = [str(limbs[top - 1])] + [str(limbs[i]).zfill(x.base_exp) for i in range(top - 2, -1, -1)]
    return "".join(parts).encode()


def convolve_mod_p(p: int, n: int, x, y=None, ctx: Context | None = None) -> np.ndarray:
    return (ctx or default_context()).convolve_mod_p(p, n, x, y)


def forward_transform(p: int, a, ctx: Context | None = None, six_step_threshold: int = 0) -> np.ndarray:
    return (ctx or default_context()).forward_transform(p, a, six_step_threshold)


def inverse_transform(p: int, a, ctx: Context | None = None, six_step_threshold: int = 0) -> np.ndarray:
    return (ctx or default_context()).inverse_transform(p, a, six_step_threshold)


def pointwise_product(p: int, a, b=None, ctx: Context | None = None) -> np.ndarray:
    return (ctx or default_context()).pointwise_product(p, a, b)


def transpose_square_sub(a, n: int, stride: int, ctx: Context | None = None) -> np.ndarray:
    return (ctx or default_context()).transpose_square_sub(a, n, stride)


def transpose_n_x_2n(a, n: int, ctx: Context | None = None) -> np.ndarray:
    return (ctx or default_context()).transpose_n_x_2n(a, n)


def transpose_2n_x_n(a, n: int, ctx: Context | None = None) -> np.ndarray:
    return (ctx or default_context()).transpose_2n_x_n(a, n)
