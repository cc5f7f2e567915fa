"""Pin the oracle (plain-C restatement, oracle/decmul_oracle.c) before trusting it:
against the reference's own known-answer tests and against the compiled
reference (golden fixtures from tests/golden/make_golden.py and, where present,
oracle/_ref live). CPU only."""
import hashlib
import os

import numpy as np
import pytest

import oracle
from paper_2011_11524_b200 import inputs

P1, P2 = oracle.P1, oracle.P2


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_make_ctx_golden(port, golden):
    for p, want in golden["kat"]["make_ctx"].items():
        assert list(port.make_ctx(int(p))) == want


def test_dif_hand_example_and_table(port, golden):
    # test_ntt.cpp:23-37 / :81-88 (p = 17, n = 4, root = 4; 2^64 = 1 mod 17)
    fwd, inv = port.ntt_plan_root(17, 4, 4)
    assert list(fwd) == golden["kat"]["ntt_table_p17_n4_root4"]["fwd"]
    assert list(inv) == golden["kat"]["ntt_table_p17_n4_root4"]["inv"]
    for x, want in golden["kat"]["dif_p17_n4_root4"]:
        assert list(port.dif_forward_root(17, x, 4)) == want


@pytest.mark.parametrize("p", [17, 97, 193, P1, P2])
def test_dif_is_bitreversed_naive_dft(port, p):
    rng = np.random.default_rng(41)
    n = 1
    while n <= 64:
        if n > 1 and (p - 1) % n:
            break
        x = rng.integers(0, p, n, dtype=np.uint64) if p < 2**62 else port.gen_residues(n, n, p)
        got = port.dif_forward(p, x)
        if n > 1:
            root = port.primitive_root(p, n)
            spec = port.naive_dft(x, root, p)
            lg = n.bit_length() - 1
            want = [spec[int(format(k, f"0{lg}b")[::-1], 2)] for k in range(n)]
            assert list(got) == [int(v) for v in want]
        n *= 2


def test_dit_undoes_dif(port):
    for p in (P1, P2):
        for n in (2, 4, 64, 1024):
            x = port.gen_residues(n, n, p)
            a = port.dit_inverse(p, port.dif_forward(p, x))
            assert [int(v) for v in a] == [int(v) * n % p for v in x]


def test_plans_match_reference(port, golden):
    for key, want in golden["ref"]["plans"].items():
        p, n = map(int, key.split(":"))
        got = port.conv_plan_info(p, n)
        for f in ("shape", "root", "psi", "psi_prime", "n1", "n2"):
            assert got[f] == want[f], (key, f)


def test_large_pair_is_reference_search(port, golden):
    assert sorted(port.find_primes(64, 30, 2)) == sorted(golden["ref"]["large_pair"])
    assert sorted(port.find_primes(64, 24, 2)) == [P1, P2]


def test_convolution_and_forward_order_vs_reference(port, ref, golden):
    for key, want in golden["ref"]["conv"].items():
        p, n = map(int, key.split(":"))
        x = ref.random_residues(want["seed_x"], n, p)
        y = ref.random_residues(want["seed_y"], n, p)
        conv = port.convolve_mod_p(p, n, x, y)
        fwd = port.forward_transform(p, x)
        if "conv" in want:
            assert [int(v) for v in conv] == want["conv"], key
            assert [int(v) for v in fwd] == want["fwd"], key
        else:
            assert sha(conv.tobytes()) == want["conv_sha"], key
            assert sha(fwd.tobytes()) == want["fwd_sha"], key
        assert list(port.inverse_transform(p, fwd)) == list(x)


def test_convolution_vs_naive_all_shapes(port):
    for p in (97, 193, P1, P2):
        for n in (1, 2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 192):
            if n > 1 and (p - 1) % n:
                continue
            for thr in (0, 4):
                x = port.gen_residues(3 * n, n, p) if p > 2**32 else np.arange(n, dtype=np.uint64) % p
                y = port.gen_residues(5 * n, n, p) if p > 2**32 else (np.arange(n, dtype=np.uint64) * 7 + 3) % p
                assert list(port.convolve_mod_p(p, n, x, y, thr)) == list(port.naive_convolve(x, y, p))


def test_multiply_kats(port, golden):
    for a, b, z in golden["kat"]["multiply"]:
        assert port.multiply(a.encode(), b.encode()) == z.encode()
    for n in (1, 2, 17, 18, 100, 1000):
        s = b"9" * n
        assert port.multiply(s) == b"9" * (n - 1) + b"8" + b"0" * (n - 1) + b"1"


def test_products_vs_reference_hashes(port, golden):
    for d, g in golden["ref"]["products_splitmix"].items():
        z = port.multiply(inputs.gen_digits(g["seed_x"], g["nx"]), inputs.gen_digits(g["seed_y"], g["ny"]))
        assert sha(z) == g["sha"], d
    for k, h in enumerate(golden["ref"]["config2_first64_sha"][:8]):
        assert sha(port.multiply(inputs.gen_digits(2 * k, 10000), inputs.gen_digits(2 * k + 1, 10000))) == h


def test_bench_stream_golden(port, ref, golden):
    for d, g in golden["ref"]["bench_mul_stream_seed42"].items():
        x, y = ref.bench_inputs(int(d), 42)
        assert sha(x) == g["x_sha"] and sha(y) == g["y_sha"]
        assert sha(port.multiply(x, y)) == g["z_sha"]


def test_random_products_vs_reference_and_schoolbook(port, ref):
    rng = np.random.default_rng(127)
    for _ in range(150):
        nx, ny = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        x = inputs.gen_digits(int(rng.integers(1 << 40)), nx)
        y = inputs.gen_digits(int(rng.integers(1 << 40)), ny)
        z = port.multiply(x, y)
        assert z == port.schoolbook_multiply(x, y) == ref.multiply(x, y)
    x = inputs.gen_digits(9, 4211)
    y = inputs.gen_digits(10, 3999)
    want = port.schoolbook_multiply(x, y)
    for be in (0, 14, 15, 16, 17):
        assert port.multiply(x, y, forced=be) == want


def test_base_and_length_selection(port, golden):
    for need, want in golden["kat"]["smallest_supported_length"]:
        assert port.smallest_supported_length(need) == want
    for dx, dy, forced, be, ln in golden["kat"]["select_base"]:
        got = port.select_base_and_length(dx, dy, forced)
        assert be is None or got[0] == be
        assert ln is None or got[1] == ln
    for key, want in golden["ref"]["select_base"].items():
        dx, dy = map(int, key.split("x"))
        assert list(port.select_base_and_length(dx, dy)) == want
    q1, q2 = sorted(golden["ref"]["large_pair"])
    for key, want in golden["ref"]["select_base_large_pair"].items():
        dx, dy = map(int, key.split("x"))
        assert list(port.select_base_and_length(dx, dy, p1=q1, p2=q2)) == want
    with pytest.raises(oracle.OracleError) as e:
        port.select_base_and_length(400000000, 400000000)
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        port.select_base_and_length(3000000, 3000000, forced=17)
    assert e.value.code == 2


def test_per_base_caps(golden):
    prod = P1 * P2
    for be, cap in golden["kat"]["per_base_caps"].items():
        top = 10 ** int(be) - 1
        assert top * top * cap < prod <= top * top * (cap + 1)


def test_pack_to_decimal_crt_carry(port, golden):
    for s, be, limbs in golden["kat"]["pack"]:
        got = port.pack(s.encode(), be)
        assert [int(v) for v in got] == limbs
        assert port.to_decimal(got, be) == s.encode()
    for a1, a2, m in golden["kat"]["crt_13_17"]:
        assert port.crt2(13, 17, a1, a2) == m
    rng = np.random.default_rng(113)
    for _ in range(1000):
        m = int(rng.integers(0, 2**63)) * int(rng.integers(1, 2**62)) % (P1 * P2)
        assert port.crt2(P1, P2, m % P1, m % P2) == m
    c = golden["kat"]["carry"]
    assert [int(v) for v in port.recover_digits(c["coeffs"], c["base_exp"], c["min_limbs"])] == c["limbs"]
    with pytest.raises(oracle.OracleError):
        port.recover_digits([82], 1, 1)  # > (B-1)^2 min_limbs (test_decimal.cpp:250-252)


def test_transposes(port, ref, golden):
    a, want = golden["kat"]["transpose_n_x_2n_2"]
    assert list(port.transpose_n_x_2n(a, 2)) == want
    a, want = golden["kat"]["transpose_2n_x_n_2"]
    assert list(port.transpose_2n_x_n(a, 2)) == want
    rng = np.random.default_rng(29)
    for n in range(1, 40, 7):
        m = rng.integers(0, 2**63, 2 * n * n, dtype=np.uint64)
        assert np.array_equal(port.transpose_n_x_2n(m, n), ref.transpose_n_x_2n(m, n))
        assert np.array_equal(port.transpose_2n_x_n(m, n), ref.transpose_2n_x_n(m, n))
        assert np.array_equal(port.transpose_2n_x_n(port.transpose_n_x_2n(m, n), n), m)
    sq = rng.integers(0, 2**63, 32 * 64, dtype=np.uint64)
    assert np.array_equal(port.transpose_square_sub(sq[32:], 32, 64), ref.transpose_square_sub(sq[32:], 32, 64))


def test_residue_fingerprint(port):
    x = inputs.gen_digits(1, 5000)
    y = inputs.gen_digits(2, 4000)
    z = port.multiply(x, y)
    for q in (2**61 - 1, 1000000007, 998244353):
        assert port.residue_mod(z, q) == port.residue_mod(x, q) * port.residue_mod(y, q) % q
        assert port.residue_mod(x[:4000], q) == int(x[:4000]) % q


def test_composed_reference_oracle_small(port, ref):
    """the composed-reference oracle (chunk products by the reference's
    multiply, exact shifted decimal sum) equals the reference's direct product; it is how
    the config-4 golden (tests/golden/golden_large.json) is made beyond the reference's cap."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_golden_large import composed_product

    for (sx, nx), (sy, ny), k in (((7, 200_003), (8, 100_001), 30_001), ((9, 5_000), (10, 4_999), 997)):
        x, y = port.gen_digits(sx, nx), port.gen_digits(sy, ny)
        assert composed_product(port, ref, x, y, k, 4) == ref.multiply(x, y)
    nines = b"9" * 20_000
    assert composed_product(port, ref, nines, nines, 3_000, 4) == b"9" * 19_999 + b"8" + b"0" * 19_999 + b"1"
