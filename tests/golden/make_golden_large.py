"""TEST INFRASTRUCTURE: exact SHA-256 goldens for BASELINE configs 3 and 4 from the
compiled reference (oracle/_ref), for tests/test_gpu_large.py.

* Config 3 (1e8 x 1e8 digits, seeds 0 and 1): the reference's own multiply (N = 2^24 is
  inside its cap).
* Config 4 (2e9 x 1e9 digits, seeds 40 and 41): beyond the reference's 3 * 2^24 cap, so by
  composition: x and y are cut into decimal chunks of K = 3.5e8 digits from
  the least significant end, every chunk product X_i * Y_j is the reference's multiply
  (run on several host threads), and the exact sum of X_i Y_j 10^(K (i + j)) is formed with
  the oracle's shifted decimal adder (or_add_shifted).

Operands come from the shared seeded generator (inputs.gen_digits / the device kernel,
pinned equal in test_host.py). Needs the compiled reference and ~90 GB of host RAM; run
once on the GPU box's host:  python tests/golden/make_golden_large.py [--threads 9]
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


def chunks(s: bytes, k: int):
    """Decimal chunks of s from the least significant end: (index, chunk without leading zeros)."""
    out, n = [], len(s)
    for i, end in enumerate(range(n, 0, -k)):
        c = s[max(0, end - k):end].lstrip(b"0")
        out.append((i, c))
    return out


def composed_product(port, ref, x: bytes, y: bytes, k: int, threads: int) -> bytes:
    xs, ys = chunks(x, k), chunks(y, k)
    pairs = [(i, j, a, b) for i, a in xs for j, b in ys if a and b]
    acc = np.zeros(len(x) + len(y) + 1, dtype=np.uint8)
    for s in range(0, len(pairs), threads):
        batch = pairs[s:s + threads]
        prods = ref.multiply_batch([p[2] for p in batch], [p[3] for p in batch], threads)
        for (i, j, _, _), z in zip(batch, prods):
            port.add_shifted(acc, z, k * (i + j))
        print(f"  chunk products {s + len(batch)}/{len(pairs)}", flush=True)
    digits = (acc[::-1] + 48).tobytes().lstrip(b"0")
    return digits or b"0"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=9)
    ap.add_argument("--out", default=os.path.join(HERE, "golden_large.json"))
    args = ap.parse_args()
    port, ref = oracle.port(), oracle.ref()
    res = {}

    # the composition itself, checked against a direct reference product
    x, y = port.gen_digits(7, 2_000_003), port.gen_digits(8, 1_000_001)
    assert composed_product(port, ref, x, y, 300_001, args.threads) == ref.multiply(x, y)

    t = time.time()
    x, y = port.gen_digits(0, 10**8), port.gen_digits(1, 10**8)
    z = ref.multiply(x, y)
    res["config3"] = dict(seeds=[0, 1], digits=[10**8, 10**8], length=len(z), sha256=hashlib.sha256(z).hexdigest(),
                          method="reference multiply")
    print("config 3", res["config3"], f"{time.time() - t:.0f} s", flush=True)
    del x, y, z

    t = time.time()
    x, y = port.gen_digits(40, 2 * 10**9), port.gen_digits(41, 10**9)
    z = composed_product(port, ref, x, y, K_CHUNK, args.threads)
    res["config4"] = dict(seeds=[40, 41], digits=[2 * 10**9, 10**9], length=len(z),
                          sha256=hashlib.sha256(z).hexdigest(), method="composed reference",
                          chunk_digits=K_CHUNK)
    print("config 4", res["config4"], f"{time.time() - t:.0f} s", flush=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
