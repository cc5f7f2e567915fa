"""The `decmul` CLI (tools/decmul_cli.cpp, reference tools/main.cpp surfaces) and the GPU
self-test (decmul_gpu_selftest, reference selftest.cpp:79-219) on the device."""
import os
import re
import subprocess

import pytest

from paper_2011_11524_b200 import inputs

pytestmark = pytest.mark.gpu
CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "decmul")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_mul_matches_reference(ref, tmp_path):
    assert run("mul", "12", "34").stdout == "408\n"
    assert run("mul", "0", "999").stdout == "0\n"
    x, y = inputs.gen_digits(3, 5000), inputs.gen_digits(4, 3000)
    r = run("mul", x.decode(), y.decode())
    assert r.returncode == 0 and r.stdout.encode() == ref.multiply(x, y) + b"\n"
    # --file: ASCII digits with an optional trailing newline (reference main.cpp:19-29)
    x, y = inputs.gen_digits(5, 200000), inputs.gen_digits(6, 150000)
    (tmp_path / "a").write_bytes(x + b"\n")
    (tmp_path / "b").write_bytes(y + b"\r\n")
    r = subprocess.run([CLI, "mul", "--file", str(tmp_path / "a"), str(tmp_path / "b")], capture_output=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout == ref.multiply(x, y) + b"\n"


def test_cli_errors_exit_1():
    r = run("mul", "012", "3")
    assert r.returncode == 1 and "error: decimal: leading zero" in r.stderr
    r = run("mul", "1x", "3")
    assert r.returncode == 1 and "error: decimal: non-digit character" in r.stderr
    r = run("mul", "--file", "/nonexistent/a", "/nonexistent/b")
    assert r.returncode == 1 and "cannot open file" in r.stderr


def test_cli_bench_mul_key_values():
    r = run("bench", "mul", "--digits", "10000", "--digits", "1000000", "--iters", "3")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 2
    kv = [dict(re.findall(r"(\w+)=(\S+)", ln)) for ln in lines]
    assert kv[0]["bench"] == "mul" and kv[0]["base_exp"] == "17" and kv[0]["length"] == "1536"
    assert kv[1]["base_exp"] == "16" and kv[1]["length"] == str(1 << 17) and kv[1]["iters"] == "3"
    assert all(int(k["product_digits"]) in (2 * int(k["digits"]), 2 * int(k["digits"]) - 1) for k in kv)
    assert all(float(k["seconds_per_mul"]) > 0 for k in kv)
    for variant in ("shoup", "montgomery", "solinas"):
        r = run("bench", "modmul", "--variant", variant)
        assert r.returncode == 0 and float(re.search(r"modmuls_per_second=(\S+)", r.stdout).group(1)) > 1e10


def test_selftest_passes_and_detects_injected_fault(gpu):
    r = run("selftest")
    assert r.returncode == 0, r.stdout
    suites = re.findall(r"suite=(\w+) checks=(\d+) failures=(\d+)", r.stdout)
    assert [s[0] for s in suites] == ["field_identities", "transform_roundtrip", "convolution_vs_direct",
                                      "crt_recompose", "base_division", "carry_recovery", "small_products"]
    assert all(int(c) > 0 and f == "0" for _, c, f in suites)
    assert int(dict((n, c) for n, c, _ in suites)["field_identities"]) == 4 * (200 * 5 + 1)
    assert r.stdout.strip().endswith("selftest_failures=0")
    r = run("selftest", "--inject-fault")
    assert r.returncode == 1
    assert "suite=fault_injection checks=2 failures=2" in r.stdout
    # the corrupted entry was restored: the context still passes afterwards
    f, report = gpu.selftest(inject_fault=True)
    assert f == 2 and "suite=small_products checks=" in report
    f, report = gpu.selftest()
    assert f == 0, report
