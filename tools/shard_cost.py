#!/usr/bin/env python3
"""In-library sharded product vs the unsharded one through the host API (decmul_gpu_multiply /
decmul_gpu_multiply_sharded on pinned-free host bytes), G ranks sharing this box's GPUs.
    python tools/shard_cost.py --nx 2000000000 --ny 1000000000 --ranks 1 2"""
import argparse
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_11524_b200 as dm  # noqa: E402
from paper_2011_11524_b200 import inputs  # noqa: E402


def timed(f, reps):
    best, out = 1e30, None
    for _ in range(reps):
        t = time.perf_counter()
        out = f()
        best = min(best, time.perf_counter() - t)
    return best * 1e3, out


def pinned(b: bytes):
    import numpy as np
    import torch

    t = torch.empty(len(b), dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = np.frombuffer(b, dtype=np.uint8)
    return t


def call(ctx, name, x, y, out):
    import ctypes as C

    n = C.c_size_t()
    args = [C.c_void_p(x.data_ptr()), C.c_size_t(x.numel()), C.c_void_p(y.data_ptr()), C.c_size_t(y.numel()),
            C.c_void_p(out.data_ptr()), C.c_size_t(out.numel()), C.byref(n)]
    if name == "decmul_gpu_multiply":
        args += [C.c_uint(0), C.c_int(0)]
    else:
        args += [C.c_int(0)]
    ctx._call(name, *args)
    return n.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=2_000_000_000)
    ap.add_argument("--ny", type=int, default=1_000_000_000)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    x, y = pinned(inputs.gen_digits(40, a.nx)), pinned(inputs.gen_digits(41, a.ny))
    out = torch.empty(a.nx + a.ny + 1, dtype=torch.uint8, pin_memory=True)
    ctx = dm.Context(0)
    ms, n = timed(lambda: call(ctx, "decmul_gpu_multiply", x, y, out), a.reps)
    ref = hashlib.sha256(out.numpy()[:n].tobytes()).hexdigest()
    print(f"unsharded: {ms:.1f} ms (host API from pinned buffers, wall, best of {a.reps})", flush=True)
    ctx.close()
    for G in a.ranks:
        c = dm.Context(devices=[0] * G)
        ms_g, ng = timed(lambda: call(c, "decmul_gpu_multiply_sharded", x, y, out), a.reps)
        same = hashlib.sha256(out.numpy()[:ng].tobytes()).hexdigest() == ref
        print(f"sharded G={G} (ranks sharing GPU 0): {ms_g:.1f} ms, x{ms_g / ms:.3f} of unsharded, "
              f"same digits: {same}", flush=True)
        c.close()


if __name__ == "__main__":
    main()
