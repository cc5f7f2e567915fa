"""Sharded large products on one GPU: all G shards run sequentially in one process
(LocalComm), so every device step of the multi-GPU path (column/row-sharded passes,
block reorders, distributed carry) is exercised bit-exactly without ranks waiting on
each other. The NCCL transport is the same sequence with torch.distributed."""
import os

import pytest

import paper_2011_11524_b200 as dm
from paper_2011_11524_b200 import inputs
from paper_2011_11524_b200.sharded import DeviceBackend, LocalComm, sharded_multiply

pytestmark = pytest.mark.gpu


def _run(gpu, G, hx, hy, squaring=False):
    import torch

    be = DeviceBackend(gpu)
    plan = be.plan(len(hx), len(hy), G)
    x = torch.frombuffer(bytearray(hx), dtype=torch.uint8).cuda()
    y = x if squaring else torch.frombuffer(bytearray(hy), dtype=torch.uint8).cuda()
    out = torch.zeros(len(hx) + len(hy), dtype=torch.uint8, device="cuda")
    n = sharded_multiply(be, LocalComm(G), plan, list(range(G)), [x] * G, [y] * G, [out] * G, squaring=squaring)
    torch.cuda.synchronize()
    return bytes(out[:n].cpu().numpy()), plan


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nx,ny", [(300000, 250000), (1000000, 999999), (2000000, 700000)])
def test_sharded_matches_reference(gpu, ref, G, nx, ny):
    hx, hy = inputs.gen_digits(nx + G, nx), inputs.gen_digits(ny + 7 * G, ny)
    z, plan = _run(gpu, G, hx, hy)
    assert plan.ranks == G and plan.local_len * G == plan.length
    assert z == ref.multiply(hx, hy)


@pytest.mark.parametrize("G", [2, 8])
def test_sharded_squaring_and_nines(gpu, G):
    n = 400000
    z, _ = _run(gpu, G, b"9" * n, b"9" * n, squaring=True)
    assert z == b"9" * (n - 1) + b"8" + b"0" * (n - 1) + b"1"


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_large_pair_radix3_columns(gpu, ref, G):
    """The q-pair's 3 * 2^k lengths put the radix-3 pass in the column phase (K = 2)."""
    os.environ["DECMUL_FORCE_LARGE_PAIR"] = "1"
    try:
        hx, hy = inputs.gen_digits(5, 600000), inputs.gen_digits(6, 500000)
        z, plan = _run(gpu, G, hx, hy)
        assert plan.p1 == dm.Q1 and plan.col_passes == 2
    finally:
        del os.environ["DECMUL_FORCE_LARGE_PAIR"]
    assert z == ref.multiply(hx, hy)


def test_nccl_transport_single_rank(gpu, ref):
    """The TorchComm path over a real NCCL process group (all_to_all_single,
    all_gather_object) — world size 1, the only NCCL group one GPU can host."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2011_11524_b200.sharded import TorchComm, rank_digit_range

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        be = DeviceBackend(gpu)
        hx, hy = inputs.gen_digits(41, 900000), inputs.gen_digits(42, 800000)
        plan = be.plan(len(hx), len(hy), 1)
        x = torch.frombuffer(bytearray(hx), dtype=torch.uint8).cuda()
        y = torch.frombuffer(bytearray(hy), dtype=torch.uint8).cuda()
        out = torch.zeros(len(hx) + len(hy), dtype=torch.uint8, device="cuda")
        n = sharded_multiply(be, TorchComm(dist), plan, [0], [x], [y], [out])
        torch.cuda.synchronize()
        assert rank_digit_range(plan, 0, n) == (0, n)
        assert bytes(out[:n].cpu().numpy()) == ref.multiply(hx, hy)
    finally:
        dist.destroy_process_group()
