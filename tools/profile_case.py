"""Short, fixed launch sequence of one bench workload, for ncu (never timed for the bench).

    python tools/profile_case.py --config 2 --reps 3
"""
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--digits", type=int, default=0, help="override both operand sizes (single products)")
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.digits:
        cfg.update(nx=a.digits, ny=a.digits)
    ctx = dm.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    sp = s.cuda_stream
    count, nx, ny = cfg["count"], cfg["nx"], cfg["ny"]
    (sx, sy), (mx, my) = cfg["seeds"], cfg["modes"]
    mode = 1 if cfg["modes"] == (1, 1) else 0
    xs = torch.empty(count * nx, dtype=torch.uint8, device="cuda")
    ys = torch.empty(count * ny, dtype=torch.uint8, device="cuda")
    outs = torch.empty(count * (nx + ny), dtype=torch.uint8, device="cuda")
    lens = torch.zeros(count, dtype=torch.int64, device="cuda")
    if count > 1:
        ctx.generate_digits(xs.data_ptr(), nx, 0, count=count, seed_step=2, mode=mx, stream=sp)
        ctx.generate_digits(ys.data_ptr(), ny, 1, count=count, seed_step=2, mode=my, stream=sp)
    else:
        ctx.generate_digits(xs.data_ptr(), nx, sx, mode=mx, stream=sp)
        ctx.generate_digits(ys.data_ptr(), ny, sy, mode=my, stream=sp)
    for r in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if count > 1:
            ctx.multiply_batch_device(count, xs.data_ptr(), nx, ys.data_ptr(), ny, outs.data_ptr(), nx + ny,
                                      lens.data_ptr(), stream=sp)
        else:
            sq = mode == 1
            ctx.multiply_device(xs.data_ptr(), nx, xs.data_ptr() if sq else ys.data_ptr(), ny, outs.data_ptr(),
                                nx + ny, stream=sp, squaring=sq, sync=False)
        torch.cuda.synchronize()
        print(f"rep {r}: {(time.perf_counter() - t) * 1e3:.3f} ms (wall, incl. launch)")
    print(ctx.stats())


if __name__ == "__main__":
    main()
