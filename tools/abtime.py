#!/usr/bin/env python3
"""A/B device timing of library variants (tuning only; never a bench number).

    python tools/abtime.py --config 4 --rounds 3 lib_a.so lib_b.so ...

Each round runs every variant in a fresh process (alternating order), timing --steps
products of the bench workload with CUDA events and checking the product's SHA-256
against the golden; prints ms/step and the per-kernel breakdown of one profiled step."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, steps):
    sys.path.insert(0, ROOT)
    import torch

    import bench
    import paper_2011_11524_b200 as dm

    cfg = bench.CONFIGS[config]
    ctx = dm.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    sp = s.cuda_stream
    count, nx, ny = cfg["count"], cfg["nx"], cfg["ny"]
    (sx, sy), (mx, my) = cfg["seeds"], cfg["modes"]
    sq = cfg["modes"] == (1, 1)
    xs = torch.empty(count * nx, dtype=torch.uint8, device="cuda")
    ys = xs if sq else torch.empty(count * ny, dtype=torch.uint8, device="cuda")
    outs = torch.empty(count * (nx + ny), dtype=torch.uint8, device="cuda")
    lens = torch.zeros(count, dtype=torch.int64, device="cuda")
    if count > 1:
        ctx.generate_digits(xs.data_ptr(), nx, 0, count=count, seed_step=2, mode=mx, stream=sp)
        ctx.generate_digits(ys.data_ptr(), ny, 1, count=count, seed_step=2, mode=my, stream=sp)
    else:
        ctx.generate_digits(xs.data_ptr(), nx, sx, mode=mx, stream=sp)
        if not sq:
            ctx.generate_digits(ys.data_ptr(), ny, sy, mode=my, stream=sp)

    def step():
        if count > 1:
            ctx.multiply_batch_device(count, xs.data_ptr(), nx, ys.data_ptr(), ny, outs.data_ptr(), nx + ny,
                                      lens.data_ptr(), stream=sp)
        else:
            ctx.multiply_device(xs.data_ptr(), nx, ys.data_ptr(), ny, outs.data_ptr(), nx + ny, stream=sp,
                                squaring=sq, sync=False)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ok = None
    if count == 1:
        n = ctx.result_length()
        pin = torch.empty(min(n, 1 << 28), dtype=torch.uint8, pin_memory=True)
        got = bench.device_sha(outs, n, pin)
        g = bench.golden_sha(cfg)
        if g is not None:
            ok = (n, got) == (g["length"], g["sha256"])
        elif cfg.get("golden") == "nines":
            ok = (n, got) == bench.nines_square_sha(nx)
    ctx.profile(True)
    step()
    torch.cuda.synchronize()
    rep = ctx.profile_report()
    ctx.profile(False)
    agg = {}
    for name, t, _, _ in rep:
        agg[name] = agg.get(name, 0.0) + t
    print(json.dumps({"ms": ms, "ok": ok, "kernels": agg}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        return child(a.config, a.steps)
    res = {lib: [] for lib in a.libs}
    for r in range(a.rounds):
        order = a.libs if r % 2 == 0 else a.libs[::-1]
        for lib in order:
            env = dict(os.environ, DECMUL_GPU_LIB=os.path.abspath(lib))
            p = subprocess.run([sys.executable, __file__, "--child", "--config", str(a.config), "--steps",
                                str(a.steps)], capture_output=True, text=True, env=env)
            if p.returncode:
                print(lib, "FAILED", p.stderr[-2000:], flush=True)
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res[lib].append(d)
            print(f"round {r} {os.path.basename(lib)}: {d['ms']:.3f} ms ok={d['ok']}", flush=True)
    for lib, ds in res.items():
        if not ds:
            continue
        best = min(ds, key=lambda d: d["ms"])
        ks = ", ".join(f"{k} {v:.3f}" for k, v in sorted(best["kernels"].items(), key=lambda kv: -kv[1]))
        print(f"== {os.path.basename(lib)}: min {best['ms']:.3f} ms, all {[round(d['ms'], 3) for d in ds]}; {ks}")


if __name__ == "__main__":
    main()
