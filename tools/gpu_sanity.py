"""Quick end-to-end sanity run on a GPU box (development aid, not a test)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2011_11524_b200 as dm  # noqa: E402

port = oracle.port()
ref = oracle.ref()
ctx = dm.Context(0)
fails = 0


def check(name, ok):
    global fails
    print(("PASS " if ok else "FAIL ") + name, flush=True)
    fails += 0 if ok else 1


check("kat", ctx.multiply_text(b"123456789123456789", b"987654321987654321") == b"121932631356500531347203169112635269")
check("12x34", ctx.multiply_text(b"12", b"34") == b"408")
for n in [1, 2, 17, 18, 100, 1000]:
    s = b"9" * n
    check(f"nines{n}", ctx.multiply_text(s, None) == b"9" * (n - 1) + b"8" + b"0" * (n - 1) + b"1")
rng = np.random.default_rng(1)
for d in [1, 5, 17, 35, 100, 999, 5000, 20000, 50000, 100000, 300000]:
    x = port.gen_digits(d, d)
    y = port.gen_digits(d + 1000, max(1, d - 3))
    t = time.time()
    z = ctx.multiply_text(x, y)
    t1 = time.time() - t
    plan = ctx.plan(len(x), len(y))
    check(f"mul {d} N={plan['length']} one_cta={plan['one_cta']} {t1*1e3:.1f}ms", z == ref.multiply(x, y))
x, y = ref.bench_inputs(1000000, 42)
t = time.time()
z = ctx.multiply_text(x, y)
print("1e6 time", time.time() - t)
check("cfg1 hash", hashlib.sha256(z).hexdigest() == "f2a7467883b33402bbff048158591f4d371b8ceb08ff2ebc0f98b2e0dcdd5fcf")
for p in [dm.P1, dm.P2]:
    for n in [2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 96, 192, 1536, 4096, 6144, 1 << 16, 3 << 15]:
        xs = port.gen_residues(n, n, p)
        ys = port.gen_residues(n + 7, n, p)
        check(f"conv p n={n}", np.array_equal(ctx.convolve_mod_p(p, n, xs, ys), ref.convolve_mod_p(p, n, xs, ys)))
        check(f"fwd n={n}", np.array_equal(ctx.forward_transform(p, xs), ref.forward_transform(p, xs)))
        check(f"inv n={n}", np.array_equal(ctx.inverse_transform(p, xs), ref.inverse_transform(p, xs)))
xs = [port.gen_digits(i, 10000) for i in range(64)]
ys = [port.gen_digits(1000 + i, 10000) for i in range(64)]
outs = ctx.multiply_batch(b"".join(xs), b"".join(ys), 64, 10000, 10000)
check("batch64", all(outs[i] == ref.multiply(xs[i], ys[i]) for i in range(64)))
print("fails", fails)
sys.exit(1 if fails else 0)
