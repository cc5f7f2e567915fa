#!/bin/bash
# After the TMA store epilogue became the default and the overlapped path's length readback
# went to pinned memory: all GPU tests, stage trace + bench of config 4, config 3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s11_tests.log
tail -3 gpurun_out/s11_tests.log
DECMUL_OVERLAP_TRACE=1 timeout 600 python bench.py > gpurun_out/s11_b4.json 2> gpurun_out/s11_b4_trace.txt
grep overlap gpurun_out/s11_b4_trace.txt | tail -8
python -c "
import json;d=json.load(open('gpurun_out/s11_b4.json'));print(d['ms_per_step'], d['outputs_ok'], json.dumps(d['e2e'])[:400])"
for t in 2 4; do timeout 600 python bench.py --e2e-threads $t > gpurun_out/s11_b4_t$t.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s11_b4_t$t.json'));print($t, d['e2e']['ms_per_step'])"; done
timeout 600 python bench.py --config 3 > gpurun_out/s11_b3.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s11_b3.json'));print(d['ms_per_step'], json.dumps(d['e2e'])[:300])"
