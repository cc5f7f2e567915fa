"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs in the build container only (needs /root/reference to build
oracle/_ref/libdecmul_ref.so — the unmodified reference sources compiled by
oracle/Makefile). Every value below is an output of the reference's own
functions on seeded inputs, or a literal known answer from the reference's
tests (file:line cited). The GPU box never reads /root/reference; tests there
compare against this committed file.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2011_11524_b200 import inputs  # noqa: E402

P1, P2 = oracle.P1, oracle.P2


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main():
    r = oracle.ref()
    g = {}
    # ---- literal known answers from the reference's own tests ----
    g["kat"] = {
        "make_ctx": {  # test_montfield.cpp:13-23
            str(P1): [8519684594239275007, 1677721598, 2814749760395673604],
            str(P2): [8750212600316297215, 1375731710, 1892637737899524100],
        },
        "dif_p17_n4_root4": [  # test_ntt.cpp:81-88
            [[0, 1, 0, 0], [1, 16, 4, 13]], [[1, 0, 0, 0], [1, 1, 1, 1]], [[1, 1, 1, 1], [4, 0, 0, 0]]],
        "ntt_table_p17_n4_root4": {"fwd": [1, 1, 4], "inv": [1, 1, 13]},  # test_ntt.cpp:23-37
        "multiply": [  # test_decimal.cpp:272-291
            ["12", "34", "408"], ["21", "43", "903"], ["0", "999999", "0"], ["999999", "0", "0"], ["1", "1", "1"],
            ["1", "123456789", "123456789"], ["10", "10", "100"],
            ["123456789123456789", "987654321987654321", "121932631356500531347203169112635269"]],
        "per_base_caps": {"14": 8507059171, "15": 85070591, "16": 850705, "17": 8507},  # test_decimal.cpp:54-64
        "smallest_supported_length": [[1, 2], [2, 2], [3, 3], [4, 4], [5, 6], [7, 8], [13, 16], [97, 128],
                                      [129, 192], [3 << 24, 3 << 24], [(3 << 24) + 1, 0]],  # test_decimal.cpp:66-89
        "select_base": [[1, 1, 0, 17, 2], [35, 35, 0, None, 6], [144619, 144619, 0, 17, None],
                        [144620, 144620, 0, 16, None], [100000000, 17, 0, 17, None]],  # test_decimal.cpp:91-127
        "crt_13_17": [[9, 15, 100], [0, 0, 0], [12, 16, 220]],  # test_decimal.cpp:208-233
        "carry": {"coeffs": [3, 10, 8, 0], "base_exp": 1, "min_limbs": 2, "limbs": [3, 0, 9, 0]},  # :235-244
        "pack": [["12345", 14, [12345]], ["100000000000000", 14, [0, 1]], ["0", 17, [0]],
                 ["9" * 35, 17, [99999999999999999, 99999999999999999, 9]]],  # test_decimal.cpp:129-140
        "transpose_n_x_2n_2": [[1, 2, 3, 4, 5, 6, 7, 8], [1, 5, 2, 6, 3, 7, 4, 8]],  # test_transpose.cpp:93-101
        "transpose_2n_x_n_2": [[1, 2, 3, 4, 5, 6, 7, 8], [1, 3, 5, 7, 2, 4, 6, 8]],  # test_transpose.cpp:103-109
    }
    # ---- outputs of the compiled reference ----
    out = {}
    out["large_pair"] = r.find_primes(64, 30, 2)
    out["production_pair"] = r.find_primes(64, 24, 2)
    plans = {}
    for p in (P1, P2):
        for n in (2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 96, 192, 1536, 4096, 6144, 1 << 15, 1 << 16, 1 << 17, 3 << 15,
                  1 << 24):
            plans[f"{p}:{n}"] = r.conv_plan_info(p, n)
    out["plans"] = plans
    q1, q2 = sorted(out["large_pair"])
    for p in (q1, q2):
        for n in (3 << 26, 3 << 29):
            plans[f"{p}:{n}"] = r.conv_plan_info(p, n)
    out["select_base_large_pair"] = {f"{dx}x{dy}": r.select_base_and_length(dx, dy, p1=q1, p2=q2)
                                     for dx, dy in ((2 * 10**9, 10**9), (10**10, 10**10))}
    out["select_base"] = {f"{dx}x{dy}": r.select_base_and_length(dx, dy)
                          for dx, dy in ((10**6, 10**6), (10**4, 10**4), (10**8, 10**8), (3, 3), (1234, 56789))}
    conv = {}
    for p in (P1, P2):
        for n in (1, 2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 96, 192, 768, 1536):
            x = r.random_residues(1000 + n, n, p)
            y = r.random_residues(2000 + n, n, p)
            conv[f"{p}:{n}"] = {
                "seed_x": 1000 + n, "seed_y": 2000 + n,
                "conv": [int(v) for v in r.convolve_mod_p(p, n, x, y)],
                "fwd": [int(v) for v in r.forward_transform(p, x)],
            }
        for n in (1 << 16, 3 << 15):
            x = r.random_residues(1000 + n, n, p)
            y = r.random_residues(2000 + n, n, p)
            conv[f"{p}:{n}"] = {"seed_x": 1000 + n, "seed_y": 2000 + n,
                                "conv_sha": sha(r.convolve_mod_p(p, n, x, y).tobytes()),
                                "fwd_sha": sha(r.forward_transform(p, x).tobytes())}
    out["conv"] = conv
    prods = {}
    for d in (1, 17, 18, 35, 100, 999, 10000, 20000, 100000):
        x = inputs.gen_digits(d, d)
        y = inputs.gen_digits(d + 1, max(1, d - 1))
        z = r.multiply(x, y)
        prods[str(d)] = {"seed_x": d, "nx": d, "seed_y": d + 1, "ny": max(1, d - 1), "sha": sha(z), "len": len(z)}
    out["products_splitmix"] = prods
    bench = {}
    for d in (10000, 1000000):
        x, y = r.bench_inputs(d, 42)
        z = r.multiply(x, y)
        bench[str(d)] = {"x_sha": sha(x), "y_sha": sha(y), "z_sha": sha(z), "len": len(z)}
    out["bench_mul_stream_seed42"] = bench  # reference bench.cpp:107-116 stream
    # config-2 batch sample: products k = 0..63 of the bench workload (pair seeds 2k, 2k+1)
    b = []
    for k in range(64):
        z = r.multiply(inputs.gen_digits(2 * k, 10000), inputs.gen_digits(2 * k + 1, 10000))
        b.append(sha(z))
    out["config2_first64_sha"] = b
    g["ref"] = out
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
