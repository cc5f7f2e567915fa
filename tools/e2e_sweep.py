"""Time the host-buffer batch API (config 2 shape) for several pipeline chunk counts.
Usage: python tools/e2e_sweep.py [chunks ...]   (0 = the library's default schedule)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11524_b200 as dm  # noqa: E402


def main():
    chunks = [int(v) for v in sys.argv[1:]] or [1, 4, 8, 16, 32]
    ctx = dm.Context(0)
    count, nx, ny = 4096, 10**4, 10**4
    dev = torch.device("cuda", 0)
    xs = torch.empty(count * nx, dtype=torch.uint8, device=dev)
    ys = torch.empty(count * ny, dtype=torch.uint8, device=dev)
    ctx.generate_digits(xs.data_ptr(), nx, 0, count=count, seed_step=2)
    ctx.generate_digits(ys.data_ptr(), ny, 1, count=count, seed_step=2)
    torch.cuda.synchronize()
    hx = torch.empty(count * nx, dtype=torch.uint8, pin_memory=True)
    hy = torch.empty(count * ny, dtype=torch.uint8, pin_memory=True)
    hx.copy_(xs)
    hy.copy_(ys)
    ho = torch.empty(count * (nx + ny), dtype=torch.uint8, pin_memory=True)
    hl = torch.zeros(count, dtype=torch.int64)
    ref = None
    for c in chunks:
        if c:
            os.environ["DECMUL_PIPE_CHUNKS"] = str(c)
        else:  # 0 = the library's default schedule
            os.environ.pop("DECMUL_PIPE_CHUNKS", None)
        call = lambda: ctx.multiply_batch_ptr(count, hx.data_ptr(), nx, hy.data_ptr(), ny, ho.data_ptr(),  # noqa
                                              nx + ny, hl.data_ptr())
        for _ in range(3):
            call()
        t0 = time.perf_counter()
        for _ in range(10):
            call()
        dt = (time.perf_counter() - t0) / 10
        h = hash(bytes(ho[: 4 * (nx + ny)].numpy()))
        ref = h if ref is None else ref
        print(f"chunks={c:3d}  {dt * 1e3:7.3f} ms/step  {count * (nx + ny) / dt / 1e9:7.2f} Gdigits/s  "
              f"same={h == ref}", flush=True)


if __name__ == "__main__":
    main()
