"""§8(e) on CPU: the multi-rank driver (paper_2011_11524_b200/sharded.py) — host-only
planning through the C ABI, column/segment layouts, all-to-all chunking, block reorders
and the distributed carry (halo, all-gathered {0,1,2}-maps, top-limb probe) — run over
gloo with world_size 2 and over LocalComm with 4 shards, the device steps replaced by
tests/shard_emu.py (a CPU restatement; the GPU steps are checked in test_gpu_sharded.py).
Results must equal the oracle's product byte for byte."""
import os
import socket

import pytest
import torch

import paper_2011_11524_b200 as dm
from paper_2011_11524_b200 import inputs
from paper_2011_11524_b200.sharded import (LocalComm, ShardPlan, TorchComm, rank_carry_ins, rank_digit_range,
                                            sharded_multiply)

from shard_emu import EmuBackend

CASES = [  # (digits x, digits y, seed x, seed y): N = 4096 (radices 64,64) and 3072 (3,32,32)
    (30000, 30000, 11, 12),
    (20000, 20000, 13, 14),
]


def _run(G, shards, comm, nx, ny, x, y, squaring=False):
    be = EmuBackend()
    plan = be.plan(nx, ny, G)
    outs = [torch.zeros(nx + ny, dtype=torch.uint8) for _ in shards]
    n = sharded_multiply(be, comm, plan, shards, [x] * len(shards), [y] * len(shards), outs, squaring)
    return n, outs


def _merge(n, outs, shards, G):
    """Each shard wrote only its own limbs: OR-combine (untouched bytes are 0)."""
    acc = torch.zeros_like(outs[0])
    for o in outs:
        acc |= o
    return bytes(acc[:n].tolist())


def test_host_only_plan_through_c_abi():
    import ctypes as C

    lib = dm.load_library()
    p = ShardPlan()
    assert lib.decmul_gpu_shard_plan_create(None, C.c_size_t(2 * 10**9), C.c_size_t(10**9), C.c_int(8), C.byref(p)) == 0
    # config 4 at G = 8: radix-3 + 512 column passes, 1536 x 131072 matrix, 16384-wide column blocks
    assert (p.length, p.base_exp, p.col_passes, p.rows, p.seg_len, p.col_width) == (
        201326592, 15, 2, 1536, 131072, 16384)
    assert p.local_len * 8 == p.length and (p.p1, p.p2) == (dm.Q1, dm.Q2)  # beyond 3 * 2^24
    assert lib.decmul_gpu_shard_plan_create(None, C.c_size_t(20000), C.c_size_t(20000), C.c_int(4), C.byref(p)) != 0
    assert lib.decmul_gpu_shard_plan_create(None, C.c_size_t(20000), C.c_size_t(20000), C.c_int(3), C.byref(p)) != 0


def test_rank_carry_ins():
    # ranks: identity, "always carry 1", "pass-through +1 capped"
    ident, one = 0x24, 0b010101
    assert rank_carry_ins([ident, one, ident]) == [0, 0, 1]
    assert rank_carry_ins([one, 0b101001, ident]) == [0, 1, 2]


@pytest.mark.parametrize("nx,ny,sx,sy", CASES)
def test_local_shards_match_oracle(port, nx, ny, sx, sy):
    x, y = inputs.gen_digits(sx, nx), inputs.gen_digits(sy, ny)
    want = port.multiply(x, y)
    n, outs = _run(2, [0, 1], LocalComm(2), nx, ny, x, y)
    assert _merge(n, outs, [0, 1], 2) == want


def test_four_local_shards_nines_square(port):
    x = b"9" * 30000
    n, outs = _run(4, [0, 1, 2, 3], LocalComm(4), 30000, 30000, x, x, squaring=True)
    assert _merge(n, outs, [0, 1, 2, 3], 4) == port.multiply(x, x)
    plan = EmuBackend().plan(30000, 30000, 4)
    ranges = [rank_digit_range(plan, q, n) for q in range(4)]
    assert ranges[-1][0] == 0 and ranges[0][1] == n
    assert all(ranges[q + 1][1] == ranges[q][0] for q in range(3))  # contiguous, descending


def _gloo_worker(rank, world, port_no, q, nx, ny, sx, sy):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y = inputs.gen_digits(sx, nx), inputs.gen_digits(sy, ny)
        n, outs = _run(world, [rank], TorchComm(dist), nx, ny, x, y)
        parts = [None] * world
        dist.all_gather_object(parts, bytes(outs[0][:n].tolist()))
        if rank == 0:
            q.put((n, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nx,ny,sx,sy", CASES[1:])
def test_two_rank_gloo_sharded_product(port, nx, ny, sx, sy):
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_no = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port_no, q, nx, ny, sx, sy)) for r in range(2)]
    for p in procs:
        p.start()
    n, parts = q.get(timeout=300)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    merged = bytes(a | b for a, b in zip(*parts))
    assert merged == port.multiply(inputs.gen_digits(sx, nx), inputs.gen_digits(sy, ny))
    # each rank wrote exactly its own contiguous digit range
    plan = EmuBackend().plan(nx, ny, 2)
    for q, part in enumerate(parts):
        lo, hi = rank_digit_range(plan, q, n)
        assert all(part[lo:hi]) and not any(part[:lo]) and not any(part[hi:])
