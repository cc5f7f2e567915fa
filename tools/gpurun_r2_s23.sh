#!/bin/bash
# Coalescing leader wait limited to small batches: per-call throughput, GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
for t in 1 2 4 8 16 64; do timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 4 16; do timeout 300 tools/percall_bench --threads $t --digits 1000 --iters 2000; done
} > gpurun_out/s23_percall.txt 2>&1
cat gpurun_out/s23_percall.txt | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s23_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s23_tests.log
tail -3 gpurun_out/s23_tests.log
