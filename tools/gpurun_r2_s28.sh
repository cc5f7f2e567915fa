#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for t in 1 3; do timeout 300 python bench.py --config 2 --e2e-threads $t > gpurun_out/s28_b2_t$t.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s28_b2_t$t.json'));print('threads', $t, d['e2e']['ms_per_step'], 'single', d['e2e'].get('single_call_ms'), d['outputs_ok'], d['e2e'].get('threads_agree'))"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "concurrent or batch" 2>&1 | tail -2
