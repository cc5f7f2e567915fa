"""The multi-device context inside the library (csrc/multi.cu, decmul_gpu_create_multi):
G ranks over the devices of one process. On a one-GPU box the ranks share the GPU (the
exchange becomes local device copies), so the whole in-library sharded product — compacted
digit slices per rank, column-sharded passes, peer-copy all-to-alls ordered by events, the
distributed {0,1,2}-carry protocol and per-rank digit ranges — runs bit-exactly against the
reference without any rank waiting on another inside a kernel."""
import os

import pytest

import paper_2011_11524_b200 as dm
from paper_2011_11524_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def multi():
    ctxs = {G: dm.Context(devices=[0] * G) for G in (1, 2, 4, 8)}
    yield ctxs
    for c in ctxs.values():
        c.close()


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nx,ny", [(300000, 250000), (1000000, 999999), (2000000, 700000)])
def test_in_library_sharded_product(multi, ref, G, nx, ny):
    ctx = multi[G]
    assert ctx.devices() == [0] * G
    hx, hy = inputs.gen_digits(nx + G, nx), inputs.gen_digits(ny + 7 * G, ny)
    assert ctx.multiply_sharded(hx, hy) == ref.multiply(hx, hy)


@pytest.mark.parametrize("G", [2, 8])
def test_in_library_sharded_squaring(multi, G):
    n = 400000
    z = multi[G].multiply_sharded(b"9" * n, None)
    assert z == b"9" * (n - 1) + b"8" + b"0" * (n - 1) + b"1"


@pytest.mark.parametrize("G", [2, 4])
def test_in_library_sharded_large_pair(ref, G):
    """The large pair's 3 * 2^k lengths (radix-3 pass in the column phase), fresh contexts."""
    os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
    try:
        ctx = dm.Context(devices=[0] * G)
        hx, hy = inputs.gen_digits(5, 600000), inputs.gen_digits(6, 500000)
        z = ctx.multiply_sharded(hx, hy)
        ctx.close()
    finally:
        del os.environ["DECMUL_FORCE_LARGE_PAIR"]
    assert z == ref.multiply(hx, hy)


def test_multi_context_routes_by_size(multi, ref):
    """decmul_gpu_multiply on a 4-rank context: small products on the first device, a product
    with N >= 2^22 sharded automatically; errors keep the reference's types."""
    ctx = multi[4]
    for nx, ny in ((12, 7), (10000, 10000), (3_000_001, 2_500_000)):
        x, y = inputs.gen_digits(nx, nx), inputs.gen_digits(ny + 1, ny)
        assert ctx.multiply_text(x, y) == ref.multiply(x, y), (nx, ny)
    with pytest.raises(ValueError, match="non-digit"):
        ctx.multiply_text(b"12x" * 1_000_000, b"7" * 2_500_000)
    with pytest.raises(ValueError, match="leading zero"):
        ctx.multiply_text(b"0" + b"1" * 3_000_000, b"7" * 2_500_000)
    assert ctx.multiply_text(b"12", b"34") == b"408"


def test_multi_context_batch_fan_out(multi, golden):
    """Uniform and mixed batches split over the ranks (contiguous ranges, one host thread per
    device): the config-2 products keep the reference's hashes."""
    import hashlib

    ctx = multi[4]
    xs = b"".join(inputs.gen_digits(2 * k, 10000) for k in range(64))
    ys = b"".join(inputs.gen_digits(2 * k + 1, 10000) for k in range(64))
    outs = ctx.multiply_batch(xs, ys, 64, 10000, 10000)
    assert [hashlib.sha256(z).hexdigest() for z in outs] == golden["ref"]["config2_first64_sha"]
    mixed_x = [inputs.gen_digits(100 + k, 1000 + 37 * (k % 5)) for k in range(40)]
    mixed_y = [inputs.gen_digits(200 + k, 900 + 11 * (k % 3)) for k in range(40)]
    single = dm.Context(0)
    assert ctx.multiply_batch_mixed(mixed_x, mixed_y) == single.multiply_batch_mixed(mixed_x, mixed_y)
    single.close()


def test_block_convolution_fallback(multi, ref, monkeypatch):
    """Products past the largest transform run as a block convolution (csrc/blocked.cu; SURVEY §7
    D1; the reference throws OperandTooLarge, decimal.cpp:94-96). DECMUL_BLOCK_DIGITS forces it
    at small sizes: ragged last blocks, all-zero blocks, blocks with inner leading zeros,
    squaring by equal text, one block against many, on a one-engine and a two-engine context;
    operands are validated as a whole with the reference's messages."""
    one = dm.Context(0)
    x = bytearray(inputs.gen_digits(91, 25_013))
    y = bytearray(inputs.gen_digits(92, 9_001))
    x[5_000:12_500] = b"0" * 7_500      # whole zero blocks and leading zeros inside blocks
    y[1:3_000] = b"0" * 2_999
    x, y = bytes(x), bytes(y)
    cases = [(x, y), (y, x), (x, x), (x, b"7"), (b"9" * 10_000, b"9" * 10_000), (x, inputs.gen_digits(93, 2_999))]
    for K in ("3000", "4096", "10007"):
        monkeypatch.setenv("DECMUL_BLOCK_DIGITS", K)
        for ctx in (one, multi[2]):
            for a, b in cases:
                assert ctx.multiply_text(a, b) == ref.multiply(a, b), (K, len(a), len(b))
            assert ctx.multiply_text(x, b"0") == b"0"
            with pytest.raises(ValueError, match="non-digit"):
                ctx.multiply_text(x[:20_000] + b"x" + x[20_001:], y)
            with pytest.raises(ValueError, match="leading zero"):
                ctx.multiply_text(b"0" + x, y)
    one.close()
