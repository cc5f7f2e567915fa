#!/bin/bash
# Pageable buffers overlap only under concurrency: concurrency tests, single-call CLI timing, 3-thread per-call.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_cli.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/s21_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s21_quick.log
tail -3 gpurun_out/s21_quick.log
timeout 300 tools/decmul bench mul --digits 100000000 --iters 10
timeout 300 tools/decmul bench mul --digits 30000000 --iters 10
for t in 1 3; do timeout 200 tools/percall_bench --threads $t --digits 30000000 --iters 30; done
DECMUL_OVERLAP=0 timeout 200 tools/percall_bench --threads 3 --digits 30000000 --iters 30
