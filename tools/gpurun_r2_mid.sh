#!/bin/bash
# Mid-round check: all GPU tests, smoke, bench lines of every config, launch list of config 4.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/t_mid.log 2>&1; echo "rc=$?" >> gpurun_out/t_mid.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_mid.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_mid.log
timeout 600 python bench.py > gpurun_out/bm_default.json 2> gpurun_out/bm_default.err
for c in 2 1 3 33 5; do timeout 600 python bench.py --config $c > gpurun_out/bm$c.json 2>gpurun_out/bm$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mid_cfg4.csv python tools/profile_case.py --config 4 --reps 2 > /dev/null 2>&1
tail -2 gpurun_out/t_mid.log; tail -1 gpurun_out/smoke_mid.log
for f in gpurun_out/bm*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'][:40], round(d['ms_per_step'],4), '%.3e'%d['value'], d.get('outputs_ok'), d['roofline']['product']['frac'] if 'product' in d['roofline'] else '')"; done
