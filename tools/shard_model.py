"""Per-rank cost model of the sharded product measured on ONE GPU.

All G shards of one product run sequentially in one process (LocalComm), which is exactly
the device work of the G ranks; the exchanges are timed separately (CUDA events around
each all-to-all, here device copies). Prints, per G: the product time, the exchange
time, the per-rank compute ((total - exchange) / G) and the all-to-all bytes per rank, from
which the multi-GPU time is projected as per-rank compute + bytes / link bandwidth.

    python tools/shard_model.py [--config 4] [--ranks 1,2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_11524_b200 as dm  # noqa: E402
from paper_2011_11524_b200.sharded import DeviceBackend, LocalComm, sharded_multiply  # noqa: E402


class TimedLocalComm(LocalComm):
    def __init__(self, G, stream):
        super().__init__(G)
        self.stream = stream
        self.events = []

    def all_to_all(self, sends, recvs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        super().all_to_all(sends, recvs)
        e1.record(self.stream)
        self.events.append((e0, e1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    ctx = dm.Context(0)
    stream = torch.cuda.Stream()
    be = DeviceBackend(ctx, stream)
    nx, ny = cfg["nx"], cfg["ny"]
    x = torch.empty(nx, dtype=torch.uint8, device="cuda")
    y = torch.empty(ny, dtype=torch.uint8, device="cuda")
    ctx.generate_digits(x.data_ptr(), nx, 0)
    ctx.generate_digits(y.data_ptr(), ny, 1)
    out = torch.zeros(nx + ny, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    rows = []
    for G in (int(g) for g in args.ranks.split(",")):
        plan = be.plan(nx, ny, G)
        best = None
        for _ in range(args.reps + 1):  # first run builds plans / allocations
            comm = TimedLocalComm(G, stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            n = sharded_multiply(be, comm, plan, list(range(G)), [x] * G, [y] * G, [out] * G)
            e1.record(stream)
            torch.cuda.synchronize()
            total = e0.elapsed_time(e1)
            exch = sum(a.elapsed_time(b) for a, b in comm.events)
            if best is None or total < best[0]:
                best = (total, exch)
        total, exch = best
        words = int(plan.local_len)
        a2a_bytes = 4 * 2 * words * 8 * (G - 1) // G  # 4 exchanges x 2 primes, the off-rank part
        rows.append(dict(ranks=G, product_ms=total, exchange_ms=exch, per_rank_compute_ms=(total - exch) / G,
                         all_to_all_bytes_per_rank=a2a_bytes, digits=n))
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
