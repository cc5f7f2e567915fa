#!/bin/bash
# Single one-CTA products through the pinned gather path: GPU tests, per-call throughput, determinism.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s18_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s18_tests.log
tail -3 gpurun_out/s18_tests.log
{
for t in 1 2 4 16 64; do timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 16; do timeout 300 tools/percall_bench --threads $t --digits 1000 --iters 2000; done
for t in 1 16; do timeout 300 tools/percall_bench --threads $t --digits 100 --iters 2000; done
} > gpurun_out/s18_percall.txt 2>&1
cat gpurun_out/s18_percall.txt
timeout 600 python tools/determinism.py --reps 25 > gpurun_out/s18_determinism.txt 2>&1; tail -8 gpurun_out/s18_determinism.txt
timeout 300 python bench.py --config 1 > gpurun_out/s18_b1.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s18_b1.json'));print(d['ms_per_step'], d['e2e'])"
