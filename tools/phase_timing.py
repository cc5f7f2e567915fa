"""Per-phase cycle split of k_small (config 2) from the diagnostic build
(paper_2011_11524_b200/csrc: make PHASE_TIMING=1 OUT=tools/ab/lib_phase.so OBJDIR=/tmp/obj_phase).
Usage: cp tools/ab/lib_phase.so paper_2011_11524_b200/libdecmul_gpu.so; python tools/phase_timing.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11524_b200 as dm  # noqa: E402

NAMES = ["pack (rest)", "radix-3 fwd", "forward rows", "pointwise", "inverse", "CRT + split", "carry scan", "digits out", "pack: loads", "pack: parse x"]


def main():
    ctx = dm.Context(0)
    count, n = 4096, 10**4
    xs = torch.empty(count * n, dtype=torch.uint8, device="cuda")
    ys = torch.empty(count * n, dtype=torch.uint8, device="cuda")
    ctx.generate_digits(xs.data_ptr(), n, 0, count=count, seed_step=2)
    ctx.generate_digits(ys.data_ptr(), n, 1, count=count, seed_step=2)
    outs = torch.empty(count * 2 * n, dtype=torch.uint8, device="cuda")
    lens = torch.zeros(count, dtype=torch.int64, device="cuda")
    lib = dm.load_library()
    buf = (C.c_ulonglong * 12)()
    for rep in range(3):
        ctx.multiply_batch_device(count, xs.data_ptr(), n, ys.data_ptr(), n, outs.data_ptr(), 2 * n, lens.data_ptr())
        torch.cuda.synchronize()
        lib.decmul_gpu_debug_phase_cycles(buf)
    tot = sum(buf)
    for name, v in zip(NAMES, buf):
        print(f"{name:14s} {v / count:12.0f} cycles/CTA  {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
