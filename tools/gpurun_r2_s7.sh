#!/bin/bash
# Session re-entry check: GPU tests, smoke, default bench line and configs 1-3 on the restored build.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s7_tests.log
tail -3 gpurun_out/s7_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s7_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s7_smoke.log
timeout 600 python bench.py > gpurun_out/s7_b4.json 2> gpurun_out/s7_b4.err
for c in 2 1 3; do timeout 900 python bench.py --config $c > gpurun_out/s7_b$c.json 2>gpurun_out/s7_b$c.err; done
cat gpurun_out/s7_b4.json | cut -c1-1500
for c in 2 1 3; do cut -c1-300 gpurun_out/s7_b$c.json; done
