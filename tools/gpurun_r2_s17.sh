#!/bin/bash
# Per-slot download rings of the overlapped path (pageable outputs): concurrency tests, per-call
# throughput of large std::string products from 1 and 3 threads.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "concurrent or pageable" > gpurun_out/s17_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s17_quick.log
tail -3 gpurun_out/s17_quick.log
{
for t in 1 3; do timeout 200 tools/percall_bench --threads $t --digits 100000000 --iters 10; done
for t in 1 3 6; do timeout 200 tools/percall_bench --threads $t --digits 30000000 --iters 30; done
for t in 3; do DECMUL_OVERLAP=0 timeout 200 tools/percall_bench --threads $t --digits 30000000 --iters 30; done
} > gpurun_out/s17_percall.txt 2>&1
cat gpurun_out/s17_percall.txt
