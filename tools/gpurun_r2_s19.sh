#!/bin/bash
# After the one-synchronisation readback of multiply_host: GPU tests, configs 1 / 3 / 4 bench lines.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s19_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s19_tests.log
tail -3 gpurun_out/s19_tests.log
for c in 1 3 4; do timeout 600 python bench.py --config $c > gpurun_out/s19_b$c.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s19_b$c.json'));print($c, d['ms_per_step'], d['outputs_ok'], {k:v for k,v in d['e2e'].items() if k!='note'})"; done
timeout 300 tools/percall_bench --threads 1 --digits 1000000 --iters 300
timeout 300 tools/decmul bench mul --digits 1000000 --digits 100000000 --iters 5
