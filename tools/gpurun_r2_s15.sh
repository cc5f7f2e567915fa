#!/bin/bash
# Per-call throughput again after decmul_gpu_multiply_ex (the drop-in's entry point) shares the
# coalescing / overlapped path; C++ drop-in test; compute-sanitizer availability probe.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
for t in 1 4 16 64; do timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 16; do DECMUL_COALESCE=0 timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 16; do timeout 300 tools/percall_bench --threads $t --digits 1000 --iters 2000; done
} > gpurun_out/s15_percall.txt 2>&1
cat gpurun_out/s15_percall.txt
timeout 600 python -m pytest tests/test_gpu_cpp.py tests/test_gpu_cli.py -x -q -p no:cacheprovider --timeout=300 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s15_sanitizer.txt 2>&1; echo "rc=$?" >> gpurun_out/s15_sanitizer.txt
tail -5 gpurun_out/s15_sanitizer.txt
