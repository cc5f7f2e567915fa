#!/bin/bash
# Final check of the round: all GPU tests, smoke, default bench line and reference arm.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s29_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s29_tests.log
tail -3 gpurun_out/s29_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s29_b4.json 2> gpurun_out/s29_b4.err; python -c "
import json;d=json.load(open('gpurun_out/s29_b4.json'));print(d['ms_per_step'], d['outputs_ok'], d['roofline']['product']['frac'], {k:v for k,v in d['e2e'].items() if k!='note'}, d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 | cut -c1-400
