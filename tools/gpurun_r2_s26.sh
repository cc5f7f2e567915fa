#!/bin/bash
# Cross-call overlap of pinned batches: tests, config-2 bench with 1 / 2 / 3 e2e threads.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "concurrent or batch" > gpurun_out/s26_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s26_quick.log
tail -5 gpurun_out/s26_quick.log
grep -q "rc=0" gpurun_out/s26_quick.log || exit 1
for t in 1 2 3 4; do timeout 300 python bench.py --config 2 --e2e-threads $t > gpurun_out/s26_b2_t$t.json 2>gpurun_out/s26_b2_t$t.err; python -c "
import json;d=json.load(open('gpurun_out/s26_b2_t$t.json'));print($t, d['ms_per_step'], d['outputs_ok'], {k:v for k,v in d['e2e'].items() if k!='note'})" || tail -3 gpurun_out/s26_b2_t$t.err; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s26_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s26_tests.log
tail -3 gpurun_out/s26_tests.log
