#!/bin/bash
# Small-batch path (one partial wave: no chunking; pinned gather for coalesced calls) and the
# overlapped path's staging rings for pageable buffers: GPU tests, per-call throughput, C++ bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s16_tests.log
tail -3 gpurun_out/s16_tests.log
{
for t in 1 4 16 64; do timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 16; do timeout 300 tools/percall_bench --threads $t --digits 1000 --iters 2000; done
for t in 1 3; do timeout 300 tools/percall_bench --threads $t --digits 100000000 --iters 10; done
for t in 1 3; do timeout 300 tools/percall_bench --threads $t --digits 10000000 --iters 40; done
} > gpurun_out/s16_percall.txt 2>&1
cat gpurun_out/s16_percall.txt
timeout 300 python bench.py --config 2 > gpurun_out/s16_b2.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s16_b2.json'));print(d['ms_per_step'], d['e2e'])"
