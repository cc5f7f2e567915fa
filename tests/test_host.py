"""Host-side tests (CPU only): the C-ABI library loads and exports every symbol
include/decmul_gpu.h declares, the host planner behind the C ABI matches the
reference, the Python mirror's validation/error behaviour, the workload
generator, the bench's algorithmic counts, and the N>1 sharding path over gloo."""
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2011_11524_b200 as dm
from paper_2011_11524_b200 import inputs, shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "decmul_gpu.h")) as f:
        return sorted(set(re.findall(r"\b(decmul_gpu_\w+)\s*\(", f.read())))


def test_library_exports_every_declared_symbol():
    lib = dm.load_library()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(dm.EXPORTED_SYMBOLS) == declared


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {dm.lib_path()} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dm.CudaError):
        dm.Context(0)


def test_cli_usage_errors_and_no_gpu_failure():
    """tools/decmul: malformed invocations exit 1 with "error: ..." (reference
    main.cpp:150-153); without a GPU a product fails loudly instead of falling back."""
    import subprocess

    import torch

    cli = os.path.join(ROOT, "tools", "decmul")
    if not os.path.exists(cli):
        pytest.skip("CLI not built")
    for args in (["foo"], ["mul", "1"], ["bench", "mul"], ["bench", "modmul", "--variant", "x"], []):
        r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=60)
        assert r.returncode == 1 and r.stderr.startswith("error: "), args
    if not torch.cuda.is_available():
        r = subprocess.run([cli, "mul", "12", "34"], capture_output=True, text=True, timeout=60)
        assert r.returncode == 1 and r.stderr.startswith("error: ") and r.stdout == ""


def test_planner_through_c_abi_matches_reference_kats(golden):
    for need, want in golden["kat"]["smallest_supported_length"]:
        assert dm.smallest_supported_length(need) == want
    for dx, dy, forced, be, ln in golden["kat"]["select_base"]:
        bp = dm.select_base_and_length(dx, dy, forced_base_exp=forced)
        assert be is None or bp.base_exp == be
        assert ln is None or bp.length == ln
    for key, want in golden["ref"]["select_base"].items():
        dx, dy = map(int, key.split("x"))
        assert [dm.select_base_and_length(dx, dy).base_exp, dm.select_base_and_length(dx, dy).length] == want
    q1, q2 = sorted(golden["ref"]["large_pair"])
    assert (q1, q2) == (dm.Q1, dm.Q2)
    for key, want in golden["ref"]["select_base_large_pair"].items():
        dx, dy = map(int, key.split("x"))
        bp = dm.select_base_and_length(dx, dy, pair=(q1, q2))
        assert [bp.base_exp, bp.length] == want
    with pytest.raises(dm.OperandTooLarge):
        dm.select_base_and_length(400000000, 400000000)
    with pytest.raises(dm.OperandTooLarge):
        dm.select_base_and_length(3000000, 3000000, forced_base_exp=17)
    with pytest.raises(ValueError):
        dm.select_base_and_length(1, 1, forced_base_exp=18)
    with pytest.raises(ValueError):
        dm.select_base_and_length(0, 1)


def test_planner_random_sizes_vs_port(port):
    rng = np.random.default_rng(103)
    for _ in range(500):
        dx, dy = int(rng.integers(1, 200000)), int(rng.integers(1, 200000))
        bp = dm.select_base_and_length(dx, dy)
        assert (bp.base_exp, bp.length) == port.select_base_and_length(dx, dy)
    for need in list(range(1, 300)) + [int(v) for v in rng.integers(2, 1 << 26, 300)]:
        assert dm.smallest_supported_length(need) == port.smallest_supported_length(need)


def test_build_conv_plan_matches_reference_plan(port):
    """build_conv_plan(ctx, n, six_step_threshold) through the C ABI (no GPU): shape, root and
    six-step factors equal the reference restatement's plan (conv.cpp:212-271), default and
    forced thresholds (test_conv.cpp:183-196, selftest.cpp:109-118)."""
    names = ("direct", "six_step", "three_rows")
    for p in (dm.P1, dm.P2, dm.Q1, dm.Q2):
        for n in (1, 2, 3, 4, 6, 16, 48, 64, 96, 192, 768, 1 << 15, 1 << 16, 3 << 15, 1 << 20):
            for thr in (0, 2, 4, 8, 32, 1 << 10):
                got = dm.build_conv_plan(p, n, thr)
                want = port.conv_plan_info(p, n, thr)
                assert got["shape"] == names[want["shape"]], (p, n, thr)
                assert got["root"] == want["root"], (p, n, thr)
                if got["shape"] == "six_step":
                    assert (got["n1"], got["n2"]) == (want["n1"], want["n2"]), (p, n, thr)
    for bad in (0, 5, 12 * 5, 7):
        with pytest.raises(ValueError, match="length must be 2\\^k or 3\\*2\\^k"):
            dm.build_conv_plan(dm.P1, bad)
    with pytest.raises(ValueError, match="does not divide p-1"):
        dm.build_conv_plan(dm.P1, 1 << 40)


def test_decimal_number_parse_errors():
    assert dm.DecimalNumber().text() == b"0" and dm.DecimalNumber().is_zero()
    assert dm.DecimalNumber.parse("1000").digit_count() == 4
    for bad, msg in (("", "empty"), ("01", "leading zero"), ("00", "leading zero"), ("1a", "non-digit"),
                     (" 1", "non-digit"), ("-1", "non-digit"), ("1 ", "non-digit")):
        with pytest.raises(ValueError, match=msg):
            dm.DecimalNumber.parse(bad)


def test_to_decimal_host(golden):
    for s, be, limbs in golden["kat"]["pack"]:
        assert dm.to_decimal(dm.PackedOperand(be, np.array(limbs, dtype=np.uint64))) == s.encode()
    assert dm.to_decimal(dm.PackedOperand(3, np.array([5, 7], dtype=np.uint64))) == b"7005"
    assert dm.to_decimal(dm.PackedOperand(3, np.array([5, 0], dtype=np.uint64))) == b"5"
    assert dm.to_decimal(dm.PackedOperand(3, np.array([0, 0, 0], dtype=np.uint64))) == b"0"


def test_generator_matches_oracle(port):
    for seed, n in ((0, 1), (1, 17), (77, 12345), (2**40 + 3, 100000)):
        assert inputs.gen_digits(seed, n) == port.gen_digits(seed, n)
    assert inputs.gen_digits(5, 10, mode=1) == b"9" * 10
    d = np.frombuffer(inputs.gen_digits(3, 200000), dtype=np.uint8) - 48
    assert d[0] >= 1 and d.max() == 9
    assert abs(np.bincount(d, minlength=10)[1:].std() / 20000) < 0.02


def test_bench_algorithmic_counts_match_survey():
    import bench

    # SURVEY §8(d) table
    assert bench.modmuls_per_product(1536, False) == 70656
    assert abs(bench.modmuls_per_product(1 << 17, False) - 7.86e6) / 7.86e6 < 0.01
    assert abs(bench.modmuls_per_product(1 << 24, False) - 1.36e9) / 1.36e9 < 0.01
    assert abs(bench.modmuls_per_product(1 << 24, True) - 9.23e8) / 9.23e8 < 0.01
    assert bench.hbm_bytes_per_product(1 << 24, 10**8, 10**8, False, False) == 192 * (1 << 24) + 4 * 10**8


def test_shard_ranges_partition():
    world, count = 4, 16
    allk = sorted(k for r in range(world) for k in shard.batch_range(r, world, count))
    assert allk == list(range(world * count))
    assert shard.shard_seeds(1, 2, 2) == [(4, 5), (6, 7)]
    with pytest.raises(ValueError):
        shard.batch_range(2, 2, 4)


def _gloo_worker(rank, world, port_no, q):
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seeds = shard.shard_seeds(rank, world, 3)
        o = oracle.port()
        # each rank multiplies its own products with no data-path collective ...
        hashes = [hashlib.sha256(o.multiply(inputs.gen_digits(a, 300), inputs.gen_digits(b, 300))).hexdigest()
                  for a, b in seeds]
        gathered = [None] * world
        dist.all_gather_object(gathered, (seeds, hashes))
        # ... and only the timing crosses ranks (max over ranks)
        t = shard.max_over_ranks(float(rank + 1), dist)
        if rank == 0:
            q.put((gathered, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding(port):
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_no = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert t == 2.0
    seeds = [s for g in gathered for s in g[0]]
    assert seeds == [(2 * k, 2 * k + 1) for k in range(6)]
    # the sharded products equal the single-process ones
    for (a, b), h in zip(seeds, [h for g in gathered for h in g[1]]):
        z = port.multiply(inputs.gen_digits(a, 300), inputs.gen_digits(b, 300))
        assert hashlib.sha256(z).hexdigest() == h


def test_bench_reference_arm_prints_one_json_line():
    """bench.py keeps stdout for exactly one JSON line (libraries' banners go to stderr);
    beyond the reference's 3*2^24 cap the reference arm times the reference's own multiply
    on chunk pairs of the config's operands (here with small chunks to stay fast)."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "4",
                        "--steps", "1", "--ref-chunk", "200000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "digits/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["digits_x"] == 2 * 10**9


def test_bench_reference_sample_is_the_configs_operands():
    """The reference arm's chunk products are exact chunks of the config-4 operands (the
    composed-reference decomposition, cut from the least significant end)."""
    import bench

    cfg = dict(bench.CONFIGS[4], nx=10**6, ny=5 * 10**5)
    xs, ys, cores, sample = bench.reference_sample(cfg, 10**5, 4)
    x = inputs.gen_digits(40, 10**6)
    y = inputs.gen_digits(41, 5 * 10**5)
    assert cores == 4 and len(xs) == 4
    assert xs[0] == x[-10**5:].lstrip(b"0") and ys[1] == y[-2 * 10**5:-10**5].lstrip(b"0")


def test_bench_nines_closed_form():
    import bench

    n, h = bench.nines_square_sha(5)
    assert n == 10 and h == hashlib.sha256(str((10**5 - 1) ** 2).encode()).hexdigest()


def test_copy_pool_covers_every_byte():
    """The pageable <-> pinned staging copy split (csrc/hostio.cu CopyPool) over lengths
    parts * 4096 * k + r, r = 0..4, and 1..4 worker threads (no GPU needed)."""
    import subprocess

    cpp = os.path.join(ROOT, "tests", "cpp")
    subprocess.run(["make", "-s", "-C", cpp, "test_copypool"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(cpp, "test_copypool")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "failures=0" in r.stdout, r.stdout + r.stderr
