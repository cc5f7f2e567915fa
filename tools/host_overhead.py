#!/usr/bin/env python3
"""Host-side issue cost of one product vs its device time (is a small product launch-bound?).
    python tools/host_overhead.py --config 1 --steps 200"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_11524_b200 as dm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    nx, ny = cfg["nx"], cfg["ny"]
    ctx = dm.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    sp = s.cuda_stream
    xs = torch.empty(nx, dtype=torch.uint8, device="cuda")
    ys = torch.empty(ny, dtype=torch.uint8, device="cuda")
    out = torch.empty(nx + ny, dtype=torch.uint8, device="cuda")
    ctx.generate_digits(xs.data_ptr(), nx, 0, stream=sp)
    ctx.generate_digits(ys.data_ptr(), ny, 1, stream=sp)

    def step():
        ctx.multiply_device(xs.data_ptr(), nx, ys.data_ptr(), ny, out.data_ptr(), nx + ny, stream=sp, sync=False)

    for _ in range(20):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / a.steps * 1e3
    host = (t1 - t0) / a.steps * 1e6
    # the same steps with a sleep between them (GPU idle at each start): device time per product
    ts = []
    for _ in range(50):
        torch.cuda.synchronize()
        time.sleep(0.0005)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(s)
        step()
        f1.record(s)
        torch.cuda.synchronize()
        ts.append(f0.elapsed_time(f1) * 1e3)
    ts.sort()
    print(f"config {a.config}: back-to-back {dev:.1f} us/step (events), host issue {host:.1f} us/step, "
          f"isolated product {ts[len(ts) // 2]:.1f} us (median of 50)")


if __name__ == "__main__":
    main()
