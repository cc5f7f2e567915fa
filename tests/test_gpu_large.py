"""GPU parity at BASELINE.json's full sizes: the reference's own 1e6-digit bench product
(golden SHA-256), exact SHA-256 goldens of configs 3 and 4 from the compiled reference
(config 4 by the composed-reference oracle beyond the reference's cap;
tests/golden/make_golden_large.py), the all-nines closed form (10^n - 1)^2 (reference
oracle.cpp:171-180), residue fingerprints z == x y (mod q) for 61-bit primes q, the exact
low window z mod 10^K == (x mod 10^K)(y mod 10^K) mod 10^K, and the digit count."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2011_11524_b200 as dm

pytestmark = pytest.mark.gpu

FINGERPRINT_PRIMES = (2305843009213693951, 2305843009213693921, 1152921504606846883, 4611686018427387847)
GOLDEN_LARGE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_large.json")


def large_golden(key):
    with open(GOLDEN_LARGE) as f:
        return json.load(f)[key]


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_config1_reference_bench_stream(gpu, ref, golden):
    g = golden["ref"]["bench_mul_stream_seed42"]["1000000"]
    x, y = ref.bench_inputs(10**6, 42)
    assert sha(x) == g["x_sha"]
    z = gpu.multiply_text(x, y)
    assert len(z) == g["len"] and sha(z) == g["z_sha"]


def _device_product(gpu, nx, ny, seed_x, seed_y, mode=0):
    import torch

    x = torch.empty(nx, dtype=torch.uint8, device="cuda")
    gpu.generate_digits(x.data_ptr(), nx, seed_x, mode=mode)
    if mode == 1 and nx == ny:
        y = x
    else:
        y = torch.empty(ny, dtype=torch.uint8, device="cuda")
        gpu.generate_digits(y.data_ptr(), ny, seed_y, mode=mode)
    out = torch.empty(nx + ny, dtype=torch.uint8, device="cuda")
    ln = gpu.multiply_device(x.data_ptr(), nx, y.data_ptr(), ny, out.data_ptr(), nx + ny, squaring=y is x)
    return x, y, out, ln


def _check_fingerprints(port, ref, hx, hy, hz, k=20000):
    for q in FINGERPRINT_PRIMES:
        assert port.residue_mod(hz, q) == port.residue_mod(hx, q) * port.residue_mod(hy, q) % q
    lo = ref.multiply(hx[-k:].lstrip(b"0") or b"0", hy[-k:].lstrip(b"0") or b"0")
    assert hz[-k:] == lo[-k:].rjust(k, b"0")


def test_config3_all_nines_closed_form(gpu):
    n = 10**8
    x, y, out, ln = _device_product(gpu, n, n, 0, 0, mode=1)
    assert ln == 2 * n
    z = out[:ln].cpu().numpy()
    assert (z[: n - 1] == ord("9")).all() and z[n - 1] == ord("8")
    assert (z[n: 2 * n - 1] == ord("0")).all() and z[2 * n - 1] == ord("1")


def test_config3_uniform_fingerprints(gpu, port, ref):
    n = 10**8
    x, y, out, ln = _device_product(gpu, n, n, 0, 1)
    assert ln in (2 * n - 1, 2 * n)
    hx, hy, hz = bytes(x.cpu().numpy()), bytes(y.cpu().numpy()), bytes(out[:ln].cpu().numpy())
    assert hz[:1] != b"0"
    g = large_golden("config3")  # the reference's own product of the same operands
    assert g["seeds"] == [0, 1] and (len(hz), sha(hz)) == (g["length"], g["sha256"])
    _check_fingerprints(port, ref, hx, hy, hz)


def test_config3_uniform_times_nines(gpu, port, ref):
    """Non-squaring worst case at config-3 size: 1e8 uniform digits (seed 2) times 1e8 nines
    (SURVEY §8(d) cfg3), against the SHA-256 of the reference's own product
    (tests/golden/golden_large.json config3x, also equal to the closed form x 10^n - x)."""
    import torch

    n = 10**8
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    y = torch.empty(n, dtype=torch.uint8, device="cuda")
    gpu.generate_digits(x.data_ptr(), n, 2)
    gpu.generate_digits(y.data_ptr(), n, 0, mode=1)
    out = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    ln = gpu.multiply_device(x.data_ptr(), n, y.data_ptr(), n, out.data_ptr(), 2 * n)
    hx, hy, hz = bytes(x.cpu().numpy()), bytes(y.cpu().numpy()), bytes(out[:ln].cpu().numpy())
    g = large_golden("config3x")
    assert g["seeds"] == [2, "nines"] and (len(hz), sha(hz)) == (g["length"], g["sha256"])
    _check_fingerprints(port, ref, hx, hy, hz)


def test_lambda16_cap_all_nines(gpu):
    """All nines at the largest lambda = 16 size (reference acceptance.cpp:275-321, 850705 limbs)."""
    n = 850705 * 16
    x, y, out, ln = _device_product(gpu, n, n, 0, 0, mode=1)
    assert gpu.plan(n, n)["base_exp"] == 16
    z = out[:ln].cpu().numpy()
    assert ln == 2 * n and (z[: n - 1] == 57).all() and z[n - 1] == 56 and (z[n:-1] == 48).all() and z[-1] == 49


def _device_residues(port, t, qs, chunk=1 << 31):
    """Residues of a device digit tensor, streamed to the host in chunks (no full copy)."""
    res = [0] * len(qs)
    for off in range(0, t.numel(), chunk):
        a = t[off:off + chunk].cpu().numpy()
        r = port.residues(a, qs)
        res = [(res[k] * pow(10, a.size, q) + r[k]) % q for k, q in enumerate(qs)]
    return res


def _low_window(t, k):
    return bytes(t[-k:].cpu().numpy())


def test_config5_ten_billion_digits(gpu, port, ref):
    """1e10 x 1e10 digits (BASELINE config 5) on one B200: N = 3 * 2^29 under the large
    pair, 4 residue arrays of 12.9 GB. Checked against the composed-reference SHA-256
    (when tests/golden/golden_large.json holds it), streamed residue fingerprints, the
    exact low window and the digit count."""
    import torch

    n = 10**10
    plan = gpu.plan(n, n)
    assert plan["large_pair"] and plan["length"] == 3 << 29 and plan["base_exp"] == 14
    x, y, out, ln = _device_product(gpu, n, n, 50, 51)
    assert ln in (2 * n - 1, 2 * n)
    # the first power-of-two pass (R = 256, S = 2^21) uses factorised twiddle tables
    assert gpu.stats()["table_bytes"] < 4 << 30
    z = out[:ln]
    assert int(z[0]) != ord("0")
    with open(GOLDEN_LARGE) as f:
        g = json.load(f).get("config5")  # composed from 841 reference chunk products
    if g is not None:
        h = hashlib.sha256()
        for off in range(0, ln, 1 << 31):
            h.update(z[off:off + (1 << 31)].cpu().numpy().tobytes())
        assert g["seeds"] == [50, 51] and (ln, h.hexdigest()) == (g["length"], g["sha256"])
    rx, ry, rz = (_device_residues(port, t, FINGERPRINT_PRIMES) for t in (x, y, z))
    for q, a, b, c in zip(FINGERPRINT_PRIMES, rx, ry, rz):
        assert c == a * b % q
    k = 10000
    lo = ref.multiply(_low_window(x, k).lstrip(b"0") or b"0", _low_window(y, k).lstrip(b"0") or b"0")
    assert _low_window(z, k) == lo[-k:].rjust(k, b"0")
    del x, y, out, z
    torch.cuda.empty_cache()


def test_config4_unbalanced_fingerprints(gpu, port, ref):
    """2e9 x 1e9 digits: beyond the reference's 3*2^24 cap (large prime pair, N = 3*2^26)."""
    nx, ny = 2 * 10**9, 10**9
    plan = gpu.plan(nx, ny)
    assert plan["large_pair"] and plan["length"] == 3 << 26 and plan["base_exp"] == 15
    x, y, out, ln = _device_product(gpu, nx, ny, 40, 41)
    assert ln in (nx + ny - 1, nx + ny)
    hx, hy, hz = bytes(x.cpu().numpy()), bytes(y.cpu().numpy()), bytes(out[:ln].cpu().numpy())
    g = large_golden("config4")  # composed from 18 reference chunk products
    assert g["seeds"] == [40, 41] and (len(hz), sha(hz)) == (g["length"], g["sha256"])
    _check_fingerprints(port, ref, hx, hy, hz, k=10000)
