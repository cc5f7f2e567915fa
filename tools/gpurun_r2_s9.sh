#!/bin/bash
# Overlapped host products (concurrent callers): the concurrency test, all GPU tests, then the
# default bench line with 1 / 2 / 3 / 4 e2e host threads, and config 3.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
free -g | head -2 > gpurun_out/s9_mem.txt; nproc >> gpurun_out/s9_mem.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "concurrent_large or pageable" > gpurun_out/s9_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s9_quick.log
tail -5 gpurun_out/s9_quick.log
grep -q "rc=0" gpurun_out/s9_quick.log || exit 1
for t in 1 2 3 4; do timeout 600 python bench.py --e2e-threads $t > gpurun_out/s9_b4_t$t.json 2> gpurun_out/s9_b4_t$t.err; python - <<PY
import json
d=json.load(open("gpurun_out/s9_b4_t$t.json")); print($t, d["ms_per_step"], json.dumps(d["e2e"])[:700])
PY
done
timeout 600 python bench.py --config 3 > gpurun_out/s9_b3.json 2> gpurun_out/s9_b3.err; cut -c1-200 gpurun_out/s9_b3.json; python -c "
import json;d=json.load(open('gpurun_out/s9_b3.json'));print(json.dumps(d['e2e'])[:600])"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s9_tests.log
tail -3 gpurun_out/s9_tests.log
