"""Repeat products that exercise every pass-kernel shape and require identical output each
time (a race in the shared-memory staging or swizzles would show as run-to-run drift; the
parity tests check the values themselves). compute-sanitizer is unavailable on the pool.

    python tools/determinism.py [--reps 20]
"""
import argparse
import hashlib
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_11524_b200 as dm  # noqa: E402


def digits(rng, n):
    return (str(rng.randint(1, 9)) + "".join(rng.choice("0123456789") for _ in range(n - 1))).encode()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ctx = dm.Context(0)
    rng = random.Random(7)
    cases = [(10**6, 10**6), (3 * 10**6 + 17, 2 * 10**6 + 5), (12 * 10**6, 9 * 10**6 + 1), (4097, 3001)]
    bad = 0
    for nx, ny in cases:
        x, y = digits(rng, nx), digits(rng, ny)
        ref = None
        for _ in range(args.reps):
            h = hashlib.sha256(ctx.multiply_text(x, y)).hexdigest()
            ref = ref or h
            bad += h != ref
        print(f"single {nx}x{ny}: {'ok' if bad == 0 else 'DRIFT'} {ref[:16]}", flush=True)
    nx = ny = 10**4
    xs = b"".join(digits(rng, nx) for _ in range(512))
    ys = b"".join(digits(rng, ny) for _ in range(512))
    ref = None
    for _ in range(args.reps):
        h = hashlib.sha256(b"".join(ctx.multiply_batch(xs, ys, 512, nx, ny))).hexdigest()
        ref = ref or h
        bad += h != ref
    print(f"batch 512 x (1e4 x 1e4): {'ok' if bad == 0 else 'DRIFT'} {ref[:16]}")
    print("DETERMINISTIC" if bad == 0 else f"DRIFT in {bad} runs")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
