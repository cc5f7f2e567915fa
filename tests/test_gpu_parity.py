"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden outputs. Bit-exact everywhere (integer arithmetic)."""
import hashlib
import os

import numpy as np
import pytest

import paper_2011_11524_b200 as dm
from paper_2011_11524_b200 import inputs

pytestmark = pytest.mark.gpu
P1, P2 = dm.P1, dm.P2


def sha(b):
    return hashlib.sha256(b).hexdigest()


def nines_square(n):
    return b"9" * (n - 1) + b"8" + b"0" * (n - 1) + b"1"


def test_multiply_known_answers(gpu, golden):
    for a, b, z in golden["kat"]["multiply"]:
        assert dm.multiply(dm.DecimalNumber.parse(a), dm.DecimalNumber.parse(b), ctx=gpu).text() == z.encode()
    for n in (1, 2, 17, 18, 100, 1000):
        x = dm.DecimalNumber.parse(b"9" * n)
        assert dm.multiply(x, x, ctx=gpu).text() == nines_square(n)


def test_products_match_reference_hashes(gpu, golden):
    for d, g in golden["ref"]["products_splitmix"].items():
        z = gpu.multiply_text(inputs.gen_digits(g["seed_x"], g["nx"]), inputs.gen_digits(g["seed_y"], g["ny"]))
        assert len(z) == g["len"] and sha(z) == g["sha"], d


def test_random_products_vs_schoolbook(gpu, port):
    rng = np.random.default_rng(127)
    for _ in range(200):
        nx, ny = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        x = inputs.gen_digits(int(rng.integers(1 << 40)), nx)
        y = inputs.gen_digits(int(rng.integers(1 << 40)), ny)
        assert gpu.multiply_text(x, y) == port.schoolbook_multiply(x, y)
    for d in (997, 2000, 5000):
        x, y = inputs.gen_digits(d, d), inputs.gen_digits(d + 1, d - 1)
        assert gpu.multiply_text(x, y) == port.schoolbook_multiply(x, y)


@pytest.mark.parametrize("digits", [33, 34, 35, 50, 51, 67, 68, 101, 102])
def test_padding_neutrality(gpu, port, digits):
    x, y = inputs.gen_digits(digits, digits), inputs.gen_digits(digits + 99, digits)
    assert gpu.multiply_text(x, y) == port.schoolbook_multiply(x, y)


# digit counts whose transform lengths cross the one-CTA / multi-pass boundary and
# every pass-count regime: N = 3072 (one CTA) ... 3 * 2^15, 2^17
@pytest.mark.parametrize("nx,ny", [(20000, 20000), (26000, 20000), (40000, 30000), (50000, 50000),
                                   (70000, 60000), (100000, 100000), (200000, 150000), (300000, 300000),
                                   (1000000, 999999), (1, 1000000), (17, 2000000), (123457, 1)])
def test_sizes_across_engines_vs_reference(gpu, ref, nx, ny):
    x, y = inputs.gen_digits(nx + 5, nx), inputs.gen_digits(ny + 6, ny)
    assert gpu.multiply_text(x, y) == ref.multiply(x, y)


def test_squaring_paths(gpu, ref):
    for d in (1, 40, 1234, 30000, 200000):
        s = inputs.gen_digits(d * 3, d)
        want = ref.multiply(s, None)
        assert gpu.multiply_text(s, None) == want  # aliased (&x == &y)
        assert gpu.multiply_text(s, bytes(s)) == want  # equal text, distinct buffers


def test_every_forced_base(gpu, port, ref):
    """MultiplyOptions::forced_base_exp 1..17 (the reference accepts every base its planner
    admits, decimal.cpp:78-100). Below lambda = 13 a coefficient can need more than three
    base-B digits, which takes the general recovery (digit scatter + normalisation rounds)."""
    x, y = inputs.gen_digits(1, 4211), inputs.gen_digits(2, 3999)
    want = port.schoolbook_multiply(x, y)
    for be in [0] + list(range(1, 18)):
        assert gpu.multiply_text(x, y, forced_base_exp=be) == want, be
    # larger operands through the multi-pass engine, and squaring, at small bases
    for be in (1, 2, 5, 9, 12, 13):
        for nx, ny in ((60001, 50000), (200000, 150001)):
            a, b = inputs.gen_digits(nx + be, nx), inputs.gen_digits(ny + be, ny)
            assert gpu.multiply_text(a, b, forced_base_exp=be) == ref.multiply(a, b), (be, nx, ny)
        a = inputs.gen_digits(be, 30000)
        assert gpu.multiply_text(a, None, forced_base_exp=be) == ref.multiply(a, None), be
    # worst-case magnitudes: all nines at a small base
    n9 = b"9" * 20000
    for be in (1, 3, 7):
        assert gpu.multiply_text(n9, n9 + b"9", forced_base_exp=be) == ref.multiply(n9, n9 + b"9"), be


def test_large_prime_pair_path(gpu, ref):
    """The pair used beyond the reference's 3*2^24 cap, exercised at small sizes."""
    os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
    try:
        for nx, ny in ((10000, 10000), (70000, 50000), (400000, 300000)):
            assert gpu.plan(nx, ny)["p1"] == dm.Q1
            x, y = inputs.gen_digits(nx, nx), inputs.gen_digits(ny, ny)
            assert gpu.multiply_text(x, y) == ref.multiply(x, y)
    finally:
        del os.environ["DECMUL_FORCE_LARGE_PAIR"]
    assert gpu.plan(10000, 10000)["p1"] == P1


def test_lean_memory_plan(gpu, ref):
    """The HBM-lean plan of config 5 (limbs packed into the second prime's array, first
    pass split per prime, carry sums in the dead x spectrum) at small sizes, with both
    prime pairs, squaring and not, radix-3 and power-of-two lengths."""
    os.environ["DECMUL_FORCE_LEAN"] = "1"
    try:
        for large in (False, True):
            if large:
                os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
            for nx, ny in ((30000, 30000), (70000, 50000), (300001, 250000)):
                x, y = inputs.gen_digits(nx + 1, nx), inputs.gen_digits(ny + 2, ny)
                assert gpu.multiply_text(x, y) == ref.multiply(x, y), (large, nx, ny)
                assert gpu.multiply_text(x, x) == ref.multiply(x, x), (large, nx)
    finally:
        os.environ.pop("DECMUL_FORCE_LEAN", None)
        os.environ.pop("DECMUL_FORCE_LARGE_PAIR", None)


def test_factorised_pass_tables(gpu, ref):
    """Factorised inter-pass twiddles lo[f][s mod L] * hi[f][s / L] (config 5's memory plan)
    forced at small sizes for both prime pairs, every pass with S > 1, forward and inverse."""
    import paper_2011_11524_b200 as dm2

    os.environ["DECMUL_FACTOR_TABLES"] = "1"
    try:
        for large in (False, True):
            if large:
                os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
            ctx = dm2.Context(0)  # fresh plans: tables are built per context
            for nx, ny in ((70000, 50000), (300001, 250000), (1200000, 1100000)):
                x, y = inputs.gen_digits(nx + 3, nx), inputs.gen_digits(ny + 4, ny)
                assert ctx.multiply_text(x, y) == ref.multiply(x, y), (large, nx, ny)
            assert ctx.multiply_text(x, None) == ref.multiply(x, None), large
            ctx.close()
    finally:
        os.environ.pop("DECMUL_FACTOR_TABLES", None)
        os.environ.pop("DECMUL_FORCE_LARGE_PAIR", None)


def test_radix3_twiddle_tables_both_forms(ref):
    """N = 3 2^k with the radix-3 twiddles merged into pass 1 (pre-multiplied column inputs,
    per-group pass-1 tables, a 3 x R1 inverse table) and with the factorised lo * hi pair in the
    radix-3 passes (DECMUL_R3_MERGE=0), full and factorised pass tables, both prime pairs,
    squaring and not, the fused pack and carry included."""
    for merge in ("1", "0"):
        for factor in ("0", "1"):
            os.environ["DECMUL_R3_MERGE"] = merge
            os.environ["DECMUL_FACTOR_TABLES"] = factor
            try:
                for large in (False, True):
                    if large:
                        os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
                    ctx = dm.Context(0)  # fresh plans under the knobs
                    for nx, ny in ((300001, 250000), (1400000, 1200000), (5000000, 4000001)):
                        assert ctx.plan(nx, ny)["length"] % 3 == 0
                        x, y = inputs.gen_digits(nx + 3, nx), inputs.gen_digits(ny + 4, ny)
                        assert ctx.multiply_text(x, y) == ref.multiply(x, y), (merge, factor, large, nx, ny)
                        assert ctx.multiply_text(x, None) == ref.multiply(x, None), (merge, factor, large, nx)
                    ctx.close()
                    os.environ.pop("DECMUL_FORCE_LARGE_PAIR", None)
            finally:
                for k in ("DECMUL_R3_MERGE", "DECMUL_FACTOR_TABLES", "DECMUL_FORCE_LARGE_PAIR"):
                    os.environ.pop(k, None)


def test_errors_match_reference_types(gpu):
    with pytest.raises(ValueError, match="non-digit"):
        gpu.multiply_text(b"12a4" * 1000, b"5" * 100)
    with pytest.raises(ValueError, match="leading zero"):
        gpu.multiply_text(b"0123" * 1000, b"5" * 100)
    with pytest.raises(ValueError, match="empty"):
        gpu.multiply_text(b"", b"5")
    with pytest.raises(dm.OperandTooLarge):
        gpu.multiply_text(b"9" * 3000000, b"9" * 3000000, forced_base_exp=17)
    assert gpu.multiply_text(b"0", b"123") == b"0"
    # the context stays usable after errors
    assert gpu.multiply_text(b"12", b"34") == b"408"


def test_batch_api_matches_reference(gpu, golden):
    xs = b"".join(inputs.gen_digits(2 * k, 10000) for k in range(64))
    ys = b"".join(inputs.gen_digits(2 * k + 1, 10000) for k in range(64))
    outs = gpu.multiply_batch(xs, ys, 64, 10000, 10000)
    assert [sha(z) for z in outs] == golden["ref"]["config2_first64_sha"]


def test_batch_host_pipeline_ragged_chunks(gpu, ref):
    """3001 products: the host batch path uploads / computes / downloads in 7 chunks of
    whole waves (444 one-CTA products on 148 SMs) with a ragged last chunk."""
    count, n = 3001, 10000
    xs = [inputs.gen_digits(9000 + 2 * k, n) for k in range(count)]
    ys = [inputs.gen_digits(9001 + 2 * k, n) for k in range(count)]
    outs = gpu.multiply_batch(b"".join(xs), b"".join(ys), count, n, n)
    want = ref.multiply_batch(xs, ys, os.cpu_count() or 1)
    bad = [k for k in range(count) if outs[k] != want[k]]
    assert not bad, bad[:10]


def test_batch_uneven_sizes_and_pass_engine(gpu, ref):
    for nx, ny, count in ((1, 1, 5), (35, 17, 33), (3000, 1000, 40), (60000, 40000, 3)):
        xs = [inputs.gen_digits(7 * k + nx, nx) for k in range(count)]
        ys = [inputs.gen_digits(7 * k + ny + 1, ny) for k in range(count)]
        outs = gpu.multiply_batch(b"".join(xs), b"".join(ys), count, nx, ny)
        assert outs == [ref.multiply(a, b) for a, b in zip(xs, ys)]


def test_convolution_hook_vs_reference(gpu, ref, golden):
    for key, want in golden["ref"]["conv"].items():
        p, n = map(int, key.split(":"))
        x = ref.random_residues(want["seed_x"], n, p)
        y = ref.random_residues(want["seed_y"], n, p)
        got = gpu.convolve_mod_p(p, n, x, y)
        fwd = gpu.forward_transform(p, x)
        if "conv" in want:
            assert [int(v) for v in got] == want["conv"], key
            assert [int(v) for v in fwd] == want["fwd"], key
        else:
            assert sha(got.tobytes()) == want["conv_sha"], key
            assert sha(fwd.tobytes()) == want["fwd_sha"], key
        assert np.array_equal(gpu.inverse_transform(p, fwd), x), key


def test_forced_six_step_threshold_orders(gpu, port):
    """Non-default plans (reference build_conv_plan(ctx, n, six_step_threshold), test_conv.cpp:183-196,
    selftest.cpp:109-118): the forward hook returns the spectrum in the forced plan's storage
    order (conv.hpp:19-24), the inverse hook consumes it, for every shape the threshold selects."""
    for p in (P1, P2, dm.Q1):
        for n in (64, 96, 192, 1024, 3 << 9, 1 << 13, 3 << 12):
            x = port.gen_residues(n + 5, n, p)
            for thr in (2, 4, 8, 32, 1 << 10, 0):
                fwd = gpu.forward_transform(p, x, thr)
                assert np.array_equal(fwd, port.forward_transform(p, x, thr)), (p, n, thr)
                assert np.array_equal(gpu.inverse_transform(p, fwd, thr), x), (p, n, thr)
                assert np.array_equal(gpu.inverse_transform(p, port.forward_transform(p, x, thr), thr), x)


def test_tma_tile_shapes_single_prime_and_paired_operands(gpu, port, ref):
    """Full-width row tiles moved by TMA in the launches the other tests do not reach: one prime
    per launch (the convolution hook at N = 2^21 and 3 * 2^20, maps of prime 0 only) and both
    operands in one launch (products with N = 2^21 and 3 * 2^19: maps of the second operand)."""
    for p, n in ((P1, 1 << 21), (dm.Q1, 3 << 20)):
        x = port.gen_residues(n + 1, n, p)
        y = port.gen_residues(n + 2, n - 5, p)
        assert np.array_equal(gpu.convolve_mod_p(p, n, x, y), port.convolve_mod_p(p, n, x, y)), (p, n)
        assert np.array_equal(gpu.inverse_transform(p, gpu.forward_transform(p, x)), x), (p, n)
    for (nx, ny), length in (((16_000_000, 15_000_000), 1 << 21), ((12_000_000, 9_000_001), 3 << 19)):
        x, y = inputs.gen_digits(71, nx), inputs.gen_digits(72, ny)
        assert gpu.plan(nx, ny)["length"] == length
        z, want = gpu.multiply_text(x, y), ref.multiply(x, y)
        assert len(z) == len(want) and sha(z) == sha(want), (nx, ny)


def test_convolution_hook_shorter_inputs_and_squaring(gpu, port):
    for p in (P1, P2, dm.Q1, dm.Q2):
        for n in (6, 64, 1536, 1 << 14, 3 << 13):
            x = port.gen_residues(n, n // 3, p)
            y = port.gen_residues(n + 1, n // 2, p)
            xp = np.zeros(n, np.uint64)
            yp = np.zeros(n, np.uint64)
            xp[: x.size] = x
            yp[: y.size] = y
            want = port.convolve_mod_p(p, n, xp, yp)
            assert np.array_equal(gpu.convolve_mod_p(p, n, x, y), want)
            assert np.array_equal(gpu.convolve_mod_p(p, n, xp), port.convolve_mod_p(p, n, xp, None))
    with pytest.raises(ValueError):
        gpu.convolve_mod_p(P1, 8, np.ones(9, np.uint64), np.ones(8, np.uint64))
    with pytest.raises(ValueError):
        gpu.convolve_mod_p(P1, 5, np.ones(5, np.uint64), np.ones(5, np.uint64))


def test_pointwise_and_pack_hooks(gpu, port):
    for p in (P1, P2):
        a, b = port.gen_residues(1, 1000, p), port.gen_residues(2, 1000, p)
        assert np.array_equal(gpu.pointwise_product(p, a, b), port.pointwise_product(p, a, b))
        assert np.array_equal(gpu.pointwise_product(p, a), port.pointwise_product(p, a, None))
    for d in (1, 14, 15, 16, 17, 18, 1000, 123457):
        s = inputs.gen_digits(d, d)
        for be in (14, 15, 16, 17):
            assert np.array_equal(gpu.pack(s, be), port.pack(s, be))
    with pytest.raises(ValueError):
        gpu.pack(b"1", 18)


def test_recover_decimal_hook(gpu, port):
    """CRT + carry + formatting on the device, from exact convolution residues."""
    cases = [(100, 90, 0), (5000, 5000, 0), (40000, 35000, 0), (3000, 2000, 1), (3000, 2000, 6), (40000, 35000, 11)]
    for nx, ny, forced in cases:
        x, y = inputs.gen_digits(nx, nx), inputs.gen_digits(ny, ny)
        be, n = port.select_base_and_length(nx, ny, forced)
        lx, ly = port.pack(x, be), port.pack(y, be)
        r1 = port.convolve_mod_p(P1, n, lx, ly)
        r2 = port.convolve_mod_p(P2, n, lx, ly)
        z = gpu.recover_decimal(r1, r2, P1, P2, be, min(lx.size, ly.size), nx + ny)
        assert z == port.multiply(x, y)
    # corrupted residues exceed the analytic bound -> runtime_error (decimal.cpp:174-176)
    bad = np.full(64, P1 - 1, dtype=np.uint64)
    with pytest.raises(RuntimeError, match="analytic bound"):
        gpu.recover_decimal(bad, np.full(64, P2 - 5, dtype=np.uint64), P1, P2, 17, 3, 100)


def test_transpose_hooks(gpu, port, golden):
    a, want = golden["kat"]["transpose_n_x_2n_2"]
    assert list(gpu.transpose_n_x_2n(a, 2)) == want
    a, want = golden["kat"]["transpose_2n_x_n_2"]
    assert list(gpu.transpose_2n_x_n(a, 2)) == want
    rng = np.random.default_rng(29)
    for n in list(range(1, 66, 4)) + [256]:
        m = rng.integers(0, 2**63, 2 * n * n, dtype=np.uint64)
        assert np.array_equal(gpu.transpose_n_x_2n(m, n), port.transpose_n_x_2n(m, n))
        assert np.array_equal(gpu.transpose_2n_x_n(m, n), port.transpose_2n_x_n(m, n))
    for n, stride in ((3, 3), (31, 31), (33, 64), (100, 100), (128, 200)):
        m = rng.integers(0, 2**63, n * stride, dtype=np.uint64)
        assert np.array_equal(gpu.transpose_square_sub(m, n, stride), port.transpose_square_sub(m, n, stride))


def test_transpose_rho_in_place_variants(gpu, port, monkeypatch):
    """The rho permutation runs in place row by row (reference transpose.cpp:27-47: 2n words of
    scratch): rows staged in shared memory, or -- past 128 KiB per row, forced here at small n --
    in a per-CTA 2n-word global slice; more rows than CTAs (n = 700 > 296)."""
    rng = np.random.default_rng(31)
    for force in ("0", "1"):
        monkeypatch.setenv("DECMUL_RHO_GLOBAL", force)
        for n in (1, 7, 300, 700):
            m = rng.integers(0, 2**63, 2 * n * n, dtype=np.uint64)
            t = gpu.transpose_n_x_2n(m, n)
            assert np.array_equal(t, port.transpose_n_x_2n(m, n)), (force, n)
            assert np.array_equal(gpu.transpose_2n_x_n(t, n), m), (force, n)


def test_device_api_and_generator(gpu, port):
    import torch

    n = 250000
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    y = torch.empty(n - 7, dtype=torch.uint8, device="cuda")
    out = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    gpu.generate_digits(x.data_ptr(), n, 1234)
    gpu.generate_digits(y.data_ptr(), n - 7, 99)
    torch.cuda.synchronize()
    hx, hy = bytes(x.cpu().numpy()), bytes(y.cpu().numpy())
    assert hx == inputs.gen_digits(1234, n) and hy == inputs.gen_digits(99, n - 7)
    ln = gpu.multiply_device(x.data_ptr(), n, y.data_ptr(), n - 7, out.data_ptr(), 2 * n)
    assert bytes(out[:ln].cpu().numpy()) == port.multiply(hx, hy)
    # asynchronous form on torch's stream
    s = torch.cuda.current_stream().cuda_stream
    gpu.multiply_device(x.data_ptr(), n, y.data_ptr(), n - 7, out.data_ptr(), 2 * n, stream=s, sync=False)
    torch.cuda.synchronize()
    assert gpu.result_length() == ln


def test_host_api_pageable_staging(gpu, ref):
    """Large pageable host buffers (Python bytes) take the staged path of the host API:
    a ring of four 16 MB pinned slots filled and drained by the copy pool while the DMA
    engine moves the previous slot (csrc/hostio.cu). 21M x 17M digits cross several slots
    in each direction, with ragged last slots; y uploads while x is transformed."""
    x, y = inputs.gen_digits(61, 21_000_003), inputs.gen_digits(62, 17_000_011)
    z = gpu.multiply_text(x, y)
    want = ref.multiply(x, y)
    assert len(z) == len(want) and sha(z) == sha(want)
    z2 = gpu.multiply_text(x, None)  # aliased squaring: only x is staged
    assert sha(z2) == sha(ref.multiply(x, None))


def test_concurrent_large_products_overlap_transfers(gpu, ref, monkeypatch):
    """Concurrent decmul_gpu_multiply calls with large pinned buffers take the overlapped path
    (upload / compute / download stages over two buffer slots, csrc/hostio.cu): four threads,
    three products each of different operands and sizes, one aliased squaring, one thread
    hitting a non-digit. Every product equals the ordinary locked path's (DECMUL_OVERLAP=0),
    one of them the reference's."""
    import threading

    import torch

    shapes = [(9_000_001, 8_000_003), (12_000_000, 5_000_000), (8_500_000, 8_500_000), (17_000_000, 1)]
    jobs = []
    for t, (nx, ny) in enumerate(shapes):
        x = torch.frombuffer(bytearray(inputs.gen_digits(700 + t, nx)), dtype=torch.uint8).pin_memory()
        y = torch.frombuffer(bytearray(inputs.gen_digits(800 + t, ny)), dtype=torch.uint8).pin_memory()
        out = torch.empty(nx + ny, dtype=torch.uint8).pin_memory()
        jobs.append((x, y, out))
    want = []
    monkeypatch.setenv("DECMUL_OVERLAP", "0")
    for t, (x, y, out) in enumerate(jobs):
        alias = t == 2
        n = gpu.multiply_ptr(x.data_ptr(), x.numel(), (x if alias else y).data_ptr(), x.numel() if alias else y.numel(),
                             out.data_ptr(), out.numel(), alias=alias)
        want.append((n, sha(out.numpy()[:n].tobytes())))
    x0, y0 = bytes(jobs[0][0].numpy()), bytes(jobs[0][1].numpy())
    z0 = ref.multiply(x0, y0)
    assert want[0] == (len(z0), sha(z0))
    monkeypatch.setenv("DECMUL_OVERLAP", "1")
    got, errs = {}, {}

    def worker(t):
        x, y, out = jobs[t]
        alias = t == 2
        for rep in range(3):
            out.zero_()
            try:
                n = gpu.multiply_ptr(x.data_ptr(), x.numel(), (x if alias else y).data_ptr(),
                                     x.numel() if alias else y.numel(), out.data_ptr(), out.numel(), alias=alias)
                got[(t, rep)] = (n, sha(out.numpy()[:n].tobytes()))
            except Exception as e:  # noqa
                errs[(t, rep)] = e
            if t == 1 and rep == 0:
                x[12345] = ord("x")  # the second call of this thread must fail, the third succeed again
            elif t == 1 and rep == 1:
                x[12345] = ord("7")

    saved = int(jobs[1][0][12345])
    th = [threading.Thread(target=worker, args=(t,)) for t in range(len(jobs))]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert set(errs) == {(1, 1)} and isinstance(errs[(1, 1)], ValueError) and "non-digit" in str(errs[(1, 1)])
    for (t, rep), v in got.items():
        if t == 1 and rep == 2 and saved != ord("7"):
            continue  # a different operand now; checked for length only
        assert v == want[t], (t, rep)
    assert len(got) == 11


def test_concurrent_batches_overlap(gpu, ref):
    """decmul_gpu_multiply_batch from three threads with pinned buffers (1024 one-CTA products per
    call: more than two waves, so the chunked pipeline; the context lock is released once a
    batch is enqueued and the calls alternate between two buffer sets). Every call's products
    equal the reference's; a bad digit fails only its own call."""
    import threading

    import torch

    count, nx, ny = 1024, 3000, 2500
    stride = nx + ny
    jobs, want = [], []
    for t in range(3):
        xs = b"".join(inputs.gen_digits(9000 + 2 * (t * count + k), nx) for k in range(count))
        ys = b"".join(inputs.gen_digits(9001 + 2 * (t * count + k), ny) for k in range(count))
        hx = torch.frombuffer(bytearray(xs), dtype=torch.uint8).pin_memory()
        hy = torch.frombuffer(bytearray(ys), dtype=torch.uint8).pin_memory()
        ho = torch.empty(count * stride, dtype=torch.uint8).pin_memory()
        hl = torch.zeros(count, dtype=torch.int64)
        jobs.append((hx, hy, ho, hl))
        want.append([ref.multiply(xs[k * nx:(k + 1) * nx], ys[k * ny:(k + 1) * ny]) for k in range(0, count, 97)])
    fails, errs = [], {}

    def worker(t):
        hx, hy, ho, hl = jobs[t]
        for rep in range(6):
            bad = t == 1 and rep == 2
            if bad:
                hx[500 * nx + 7] = ord("x")
            try:
                ho.zero_()
                gpu.multiply_batch_ptr(count, hx.data_ptr(), nx, hy.data_ptr(), ny, ho.data_ptr(), stride, hl.data_ptr())
                o = ho.numpy()
                got = [bytes(o[k * stride:k * stride + int(hl[k])]) for k in range(0, count, 97)]
                if got != want[t]:
                    fails.append((t, rep))
            except ValueError as e:
                errs[(t, rep)] = str(e)
            if bad:
                hx[500 * nx + 7] = jobs_saved[0]

    jobs_saved = [int(jobs[1][0][500 * nx + 7])]
    th = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for h in th:
        h.start()
    for h in th:
        h.join(timeout=300)
    assert not any(h.is_alive() for h in th), "deadlock"
    assert not fails, fails
    assert list(errs) == [(1, 2)] and "non-digit" in errs[(1, 2)]


def test_mixed_concurrent_traffic(gpu, ref):
    """One context shared by threads doing different things at once: two threads of overlapped
    large pinned products, two of large pageable ones, two of small (coalesced) products, one of
    uniform batches, one of the convolution hook. Every result is checked; nothing deadlocks (lock orders: upload -> output
    slot -> context for the overlapped path, context -> queue for the coalesced one)."""
    import threading

    import torch

    nbig = 9_000_000
    bx = torch.frombuffer(bytearray(inputs.gen_digits(901, nbig)), dtype=torch.uint8).pin_memory()
    by = torch.frombuffer(bytearray(inputs.gen_digits(902, nbig)), dtype=torch.uint8).pin_memory()
    zbig = ref.multiply(bytes(bx.numpy()), bytes(by.numpy()))
    want_big = (len(zbig), sha(zbig))
    small = [(inputs.gen_digits(1000 + k, 9000 + k), inputs.gen_digits(2000 + k, 7000 + 3 * k)) for k in range(6)]
    want_small = [ref.multiply(a, b) for a, b in small]
    bxs = [inputs.gen_digits(3000 + k, 5000) for k in range(64)]
    bys = [inputs.gen_digits(4000 + k, 5000) for k in range(64)]
    want_batch = [ref.multiply(a, b) for a, b in zip(bxs, bys)]
    p, n = P1, 3 << 10
    cx, cy = ref.random_residues(5, n, p), ref.random_residues(6, n, p)
    want_conv = gpu.convolve_mod_p(p, n, cx, cy)
    fails = []

    def big():
        out = torch.empty(2 * nbig, dtype=torch.uint8).pin_memory()
        for _ in range(4):
            m = gpu.multiply_ptr(bx.data_ptr(), nbig, by.data_ptr(), nbig, out.data_ptr(), out.numel())
            if (m, sha(out.numpy()[:m].tobytes())) != want_big:
                fails.append("big")

    xb, yb = bytes(bx.numpy()), bytes(by.numpy())

    def big_pageable():  # pageable operands: the overlapped path's own staging rings
        for _ in range(3):
            if gpu.multiply_text(xb, yb) != zbig:
                fails.append("big pageable")

    def smalls():
        for rep in range(12):
            for (a, b), w in zip(small, want_small):
                if gpu.multiply_text(a, b) != w:
                    fails.append("small")

    def batches():
        for _ in range(6):
            if gpu.multiply_batch(b"".join(bxs), b"".join(bys), 64, 5000, 5000) != want_batch:
                fails.append("batch")

    def hooks():
        for _ in range(10):
            if not np.array_equal(gpu.convolve_mod_p(p, n, cx, cy), want_conv):
                fails.append("conv")

    th = [threading.Thread(target=f) for f in (big, big, big_pageable, big_pageable, smalls, smalls, batches, hooks)]
    for h in th:
        h.start()
    for h in th:
        h.join(timeout=300)
    assert not any(h.is_alive() for h in th), "deadlock"
    assert not fails, fails


def test_batch_mixed_sizes_pointer_arrays(gpu, ref):
    """decmul_gpu_multiply_batch_ptrs (the pointer-array batch of SURVEY §8(b)): repeated
    size pairs run as uniform batches, singletons one by one; results in input order."""
    shapes = [(10000, 10000)] * 7 + [(3000, 1000)] * 3 + [(60000, 40000)] * 2 + [(5, 7), (250000, 1), (1, 1)]
    xs, ys = [], []
    for k, (nx, ny) in enumerate(shapes):
        xs.append(inputs.gen_digits(500 + 2 * k, nx))
        ys.append(inputs.gen_digits(501 + 2 * k, ny))
    xs.append(b"0")
    ys.append(inputs.gen_digits(9, 12345))
    order = list(np.random.default_rng(5).permutation(len(xs)))  # interleave the groups
    xs, ys = [xs[i] for i in order], [ys[i] for i in order]
    assert gpu.multiply_batch_mixed(xs, ys) == [ref.multiply(a, b) for a, b in zip(xs, ys)]
    with pytest.raises(ValueError, match="non-digit"):
        gpu.multiply_batch_mixed([b"12", b"3x4"], [b"5", b"6"])


def test_async_error_word(gpu):
    """Errors of the asynchronous entry points land in their own stream-ordered word: the
    device batch reports bad digits at check_errors, and synchronous calls never see them."""
    import torch

    n, count = 10000, 8
    xs = torch.full((count * n,), ord("7"), dtype=torch.uint8, device="cuda")
    ys = torch.full((count * n,), ord("3"), dtype=torch.uint8, device="cuda")
    xs[5 * n + 17] = ord("x")
    outs = torch.empty(count * 2 * n, dtype=torch.uint8, device="cuda")
    lens = torch.zeros(count, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    gpu.multiply_batch_device(count, xs.data_ptr(), n, ys.data_ptr(), n, outs.data_ptr(), 2 * n, lens.data_ptr(),
                              stream=s)
    assert gpu.multiply_text(b"12", b"34") == b"408"  # a synchronous call is unaffected
    with pytest.raises(ValueError, match="non-digit"):
        gpu.check_errors(s)
    gpu.check_errors(s)  # cleared
    xs[5 * n + 17] = ord("7")
    gpu.multiply_batch_device(count, xs.data_ptr(), n, ys.data_ptr(), n, outs.data_ptr(), 2 * n, lens.data_ptr(),
                              stream=s)
    gpu.check_errors(s)
    import sys

    sys.set_int_max_str_digits(0)
    want = str(int("7" * n) * int("3" * n)).encode()
    assert bytes(outs[:int(lens[0])].cpu().numpy()) == want


def test_device_zero_short_circuit_validates(gpu):
    """multiply_device's zero short-circuit reads the digit in stream order and validates
    both operands as DecimalNumber::parse does (decimal.cpp:29-36, :193)."""
    import torch

    zero = torch.tensor([ord("0")], dtype=torch.uint8, device="cuda")
    y = torch.tensor(list(b"12345"), dtype=torch.uint8, device="cuda")
    out = torch.empty(8, dtype=torch.uint8, device="cuda")
    assert gpu.multiply_device(zero.data_ptr(), 1, y.data_ptr(), 5, out.data_ptr(), 8) == 1
    assert int(out[0]) == ord("0")
    bad = torch.tensor(list(b"12a45"), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="non-digit"):
        gpu.multiply_device(zero.data_ptr(), 1, bad.data_ptr(), 5, out.data_ptr(), 8)
    lead = torch.tensor(list(b"012"), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="leading zero"):
        gpu.multiply_device(lead.data_ptr(), 3, zero.data_ptr(), 1, out.data_ptr(), 8)
    assert gpu.multiply_text(b"12", b"34") == b"408"


def test_errors_in_fused_pack_radix3(gpu, ref):
    """Digit validation inside the pack fused with the radix-3 pass (N = 3 2^k multi-pass
    transforms): a leading zero, a non-digit anywhere, and operand lengths that leave the
    most significant limb short, against the reference."""
    n = 300001
    x, y = inputs.gen_digits(7, n), inputs.gen_digits(8, n - 2)
    assert gpu.plan(n, n - 2)["length"] % 3 == 0 and not gpu.plan(n, n - 2)["one_cta"]
    with pytest.raises(ValueError, match="leading zero"):
        gpu.multiply_text(b"0" + x[1:], y)
    for pos in (0, 17, n // 2, n - 1):
        bad = bytearray(x)
        bad[pos] = ord(":")
        with pytest.raises(ValueError, match="non-digit"):
            gpu.multiply_text(bytes(bad), y)
    for extra in range(0, 17):
        xs = x[: n - extra]
        assert gpu.multiply_text(xs, y) == ref.multiply(xs, y)
    assert gpu.multiply_text(b"12", b"34") == b"408"


def test_profile_report(gpu):
    """Per-launch profiling (decmul_gpu_profile_*): every kernel of a product appears with its
    algorithmic work, and the records clear after a report."""
    x, y = inputs.gen_digits(3, 300000), inputs.gen_digits(4, 200000)
    gpu.profile(True)
    gpu.multiply_text(x, y)
    rep = gpu.profile_report()
    gpu.profile(False)
    names = [r[0] for r in rep]
    assert names[0].startswith("k_pack") and any(nm.startswith("k_pass_fused") for nm in names)
    assert any(nm.startswith("k_carry") for nm in names)
    assert all(ms >= 0 for _, ms, _, _ in rep)
    assert sum(mm for _, _, mm, _ in rep) > 0
    assert gpu.profile_report() == []


def test_prime_pair_option(gpu, ref, port):
    """MultiplyOptions' prime pair (decmul_gpu_multiply_ex; the reference's planner takes a
    PrimePair, decimal.hpp:71-72, its multiply pins production_primes()): the reference pair,
    the large pair and another pair from the reference's own search give the same digits; a
    pair too small for the product raises OperandTooLarge like the reference's planner."""
    import paper_2011_11524_b200 as dm2

    other = tuple(sorted(port.find_primes(64, 26, 2)))
    for nx, ny in ((10000, 10000), (250001, 200000), (3_000_000, 1_000_001)):
        x, y = inputs.gen_digits(nx + 11, nx), inputs.gen_digits(ny + 12, ny)
        want = ref.multiply(x, y)
        for pair in ((P1, P2), (dm2.Q1, dm2.Q2), other):
            assert gpu.multiply_text(x, y, primes=pair) == want, (pair, nx)
    x = inputs.gen_digits(3, 50000)
    assert gpu.multiply_text(x, None, primes=other) == ref.multiply(x, None)
    with pytest.raises(ValueError, match="prime pair"):
        gpu.multiply_text(b"12", b"34", primes=(P2, P1))
    with pytest.raises(ValueError, match="prime pair"):
        gpu.multiply_text(b"12", b"34", primes=(15, P1))
    small = tuple(sorted(port.find_primes(64, 14, 2)))  # 2-adicity 14: N <= 3 * 2^14
    with pytest.raises(dm2.OperandTooLarge):
        gpu.multiply_text(b"7" * 2_000_000, b"3" * 2_000_000, primes=small)


def test_concurrent_small_multiplies_coalesce(ref):
    """decmul_gpu_multiply from 16 threads on one context: the small products are coalesced
    into shared batch launches (leader/follower), every caller gets its own exact product,
    and a bad operand fails only its own call (also when the failing caller is a follower
    while the next leader holds the context: the lock-order case that once deadlocked)."""
    import threading

    import paper_2011_11524_b200 as dm2

    ctx = dm2.Context(0)
    n_threads, per = 16, 40
    pairs = [[(inputs.gen_digits(1000 * t + 2 * k, 10000), inputs.gen_digits(1000 * t + 2 * k + 1, 9000 + t))
              for k in range(per)] for t in range(n_threads)]
    results = [[None] * per for _ in range(n_threads)]
    errors = []

    def work(t):
        try:
            for k, (x, y) in enumerate(pairs[t]):
                if k % 8 == t % 8:  # failing calls from every thread (followers' error path)
                    try:
                        ctx.multiply_text(x[:100] + b"x" + x[101:], y)
                        errors.append("no error for a bad digit")
                    except ValueError:
                        pass
                results[t][k] = ctx.multiply_text(x, y)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(t,)) for t in range(n_threads)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    assert not errors, errors
    for t in range(n_threads):
        for k in range(0, per, 7):
            x, y = pairs[t][k]
            assert results[t][k] == ref.multiply(x, y), (t, k)
    batches, products = ctx.coalesce_stats()
    assert products >= n_threads * per and batches < products
    ctx.close()
