#!/bin/bash
# Per-call throughput of the drop-in decmul::multiply from T threads (coalescing on / off), and the
# default bench line on the final build.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
{
for t in 1 4 16 64; do timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 16; do DECMUL_COALESCE=0 timeout 300 tools/percall_bench --threads $t --digits 10000 --iters 2000; done
for t in 1 4 16; do timeout 300 tools/percall_bench --threads $t --digits 1000000 --iters 300; done
} > gpurun_out/s14_percall.txt 2>&1
cat gpurun_out/s14_percall.txt
timeout 600 python bench.py > gpurun_out/s14_b4.json 2> gpurun_out/s14_b4.err
python -c "
import json;d=json.load(open('gpurun_out/s14_b4.json'));r=d['roofline'];print(d['ms_per_step'], r['traffic'], r['algorithmic_per_launch'], d['e2e']['ms_per_step'], d['outputs_ok'])"
