"""TEST INFRASTRUCTURE: exact SHA-256 goldens for BASELINE configs 1, 3, 4 and 5 from the
compiled reference (oracle/_ref), for tests/test_gpu_large.py and bench.py's output check.

* Config 1 (1e6 x 1e6 digits, seeds 0 and 1): the reference's own multiply.
* Config "3x" (1e8 uniform digits, seed 2, times 1e8 nines): the non-squaring worst case
  of SURVEY §8(d) cfg3, the reference's own multiply.

* Config 3 (1e8 x 1e8 digits, seeds 0 and 1): the reference's own multiply (N = 2^24 is
  inside its cap).
* Configs 4 (2e9 x 1e9 digits, seeds 40 and 41) and 5 (1e10 x 1e10, seeds 50 and 51):
  beyond the reference's 3 * 2^24 cap, so by composition: x and y are cut
  into decimal chunks of K = 3.5e8 digits from the least significant end, every chunk
  product X_i * Y_j is the reference's multiply (run on several host threads), and the exact
  sum of X_i Y_j 10^(K (i + j)) is formed carry-free in uint16 digit columns and carried
  once by the oracle (or_carry_u16). Config 4: 18 chunk products; config 5: 841.

Operands come from the shared seeded generator (inputs.gen_digits / the device kernel,
pinned equal in test_host.py). Needs the compiled reference and ~90 GB (configs 3, 4) or
~160 GB (config 5) of host RAM; run once on the GPU box's host:
  python tests/golden/make_golden_large.py [--threads 9] [--configs 3,4,5]
"""
import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402

K_CHUNK = 350_000_000


def chunk(s: bytes, i: int, k: int) -> bytes:
    """Decimal chunk i of s, counted from the least significant end, without leading zeros."""
    end = len(s) - i * k
    return s[max(0, end - k):end].lstrip(b"0")


def composed_product(port, ref, x: bytes, y: bytes, k: int, threads: int) -> bytes:
    """x y = sum over chunk pairs of X_i Y_j 10^(k (i + j)): every X_i Y_j is the reference's
    multiply; the digit columns are summed carry-free in uint16 (each column gets at most
    2 min(#X chunks, #Y chunks) digits, each <= 9) and
    carried once at the end (or_carry_u16)."""
    from concurrent.futures import ThreadPoolExecutor

    nxc, nyc = -(-len(x) // k), -(-len(y) // k)
    assert 2 * 9 * min(nxc, nyc) < 65536
    pairs = [(i, j) for i in range(nxc) for j in range(nyc)]
    acc = np.zeros(len(x) + len(y) + 1, dtype=np.uint16)

    def run_batch(s):  # the reference's multiply on `threads` host threads (GIL released)
        batch = [(i, j, chunk(x, i, k), chunk(y, j, k)) for i, j in pairs[s:s + threads]]
        batch = [b for b in batch if b[2] and b[3]]
        prods = ref.multiply_batch([b[2] for b in batch], [b[3] for b in batch], threads) if batch else []
        return [(i, j, z) for (i, j, _, _), z in zip(batch, prods)]

    starts = list(range(0, len(pairs), threads))
    with ThreadPoolExecutor(1) as ex:  # batch b + 1 multiplies while batch b is summed
        nxt = ex.submit(run_batch, starts[0])
        for n, s in enumerate(starts):
            done = nxt.result()
            if n + 1 < len(starts):
                nxt = ex.submit(run_batch, starts[n + 1])
            for i, j, z in done:
                d = np.frombuffer(z, dtype=np.uint8)[::-1] - np.uint8(48)  # little-endian digits
                off = k * (i + j)
                acc[off:off + d.size] += d
            print(f"  chunk products {min(s + threads, len(pairs))}/{len(pairs)}", flush=True)
    return port.carry_u16(acc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=9)
    ap.add_argument("--out", default=os.path.join(HERE, "golden_large.json"))
    ap.add_argument("--configs", default="3,4", help="comma-separated: 1, 3, 3x, 4, 5")
    args = ap.parse_args()
    todo = set(args.configs.split(","))
    port, ref = oracle.port(), oracle.ref()
    res = {}

    # the composition itself, checked against a direct reference product
    x, y = port.gen_digits(7, 2_000_003), port.gen_digits(8, 1_000_001)
    assert composed_product(port, ref, x, y, 300_001, args.threads) == ref.multiply(x, y)

    if os.path.exists(args.out):
        with open(args.out) as f:
            res = json.load(f)
    if "1" in todo:
        x, y = port.gen_digits(0, 10**6), port.gen_digits(1, 10**6)
        z = ref.multiply(x, y)
        res["config1"] = dict(seeds=[0, 1], digits=[10**6, 10**6], length=len(z),
                              sha256=hashlib.sha256(z).hexdigest(), method="reference multiply")
        print("config 1", res["config1"], flush=True)
    if "3x" in todo:
        t = time.time()
        x, y = port.gen_digits(2, 10**8), b"9" * 10**8
        z = ref.multiply(x, y)
        res["config3x"] = dict(seeds=[2, "nines"], digits=[10**8, 10**8], length=len(z),
                               sha256=hashlib.sha256(z).hexdigest(), method="reference multiply")
        print("config 3x", res["config3x"], f"{time.time() - t:.0f} s", flush=True)
        del x, y, z
    if "3" in todo:
        t = time.time()
        x, y = port.gen_digits(0, 10**8), port.gen_digits(1, 10**8)
        z = ref.multiply(x, y)
        res["config3"] = dict(seeds=[0, 1], digits=[10**8, 10**8], length=len(z),
                              sha256=hashlib.sha256(z).hexdigest(), method="reference multiply")
        print("config 3", res["config3"], f"{time.time() - t:.0f} s", flush=True)
        del x, y, z
    for cfg, (sx, sy, nx, ny) in ((4, (40, 41, 2 * 10**9, 10**9)), (5, (50, 51, 10**10, 10**10))):
        if str(cfg) not in todo:
            continue
        t = time.time()
        x, y = port.gen_digits(sx, nx), port.gen_digits(sy, ny)
        z = composed_product(port, ref, x, y, K_CHUNK, args.threads)
        del x, y
        res[f"config{cfg}"] = dict(seeds=[sx, sy], digits=[nx, ny], length=len(z),
                                   sha256=hashlib.sha256(z).hexdigest(), method="composed reference",
                                   chunk_digits=K_CHUNK)
        print(f"config {cfg}", res[f"config{cfg}"], f"{time.time() - t:.0f} s", flush=True)
        del z
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
