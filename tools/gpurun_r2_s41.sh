#!/bin/bash
# After the fused pass bulk copies and bulk store: all GPU tests, bench lines of configs 4, 3, 33, 5, 1, 2; determinism.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s41_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s41_tests.log
tail -3 gpurun_out/s41_tests.log
for c in 4 3 33 5 1 2; do timeout 900 python bench.py --config $c > gpurun_out/s41_b$c.json 2>gpurun_out/s41_b$c.err; python -c "
import json;d=json.load(open('gpurun_out/s41_b$c.json'));print($c, d['ms_per_step'], d['outputs_ok'], d['roofline']['product']['frac'], d['e2e']['ms_per_step'], d['clocks']['reasons'])"; done
timeout 600 python tools/determinism.py --reps 25 > gpurun_out/s41_determinism.txt 2>&1; tail -2 gpurun_out/s41_determinism.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s41_bench_launches_cfg4.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
