#!/bin/bash
# Coalescing leader wait A/B (per-call throughput of 1e4-digit std::string products).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
for w in 0 40 80; do for t in 1 2 4 16 64; do echo "wait_us=$w"; DECMUL_COALESCE_WAIT_US=$w timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done; done
} > gpurun_out/s22_percall.txt 2>&1
paste -d' ' - - < gpurun_out/s22_percall.txt | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "coalesce or concurrent" 2>&1 | tail -2
