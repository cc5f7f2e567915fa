#!/bin/bash
# Round-2 baseline on a GPU box: gpu tests, bench lines for every config, launch lists.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_base.log 2>&1; echo "rc=$?" >> gpurun_out/t_base.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err
for c in 2 1 3 5; do timeout 600 python bench.py --config $c > gpurun_out/b$c.json 2>gpurun_out/b$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2>gpurun_out/b_ref.err
for c in 1 2 4; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv python tools/profile_case.py --config $c --reps 2 > /dev/null 2>&1; done
ls -la gpurun_out
