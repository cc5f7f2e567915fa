#!/bin/bash
# Per-GPU shares of the config-2 batch under an even split over 1 / 2 / 4 / 8 GPUs (one B200).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for b in 4096 2048 1024 512; do timeout 300 python bench.py --config 2 --batch $b --e2e-threads 1 > gpurun_out/s36_b2_$b.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s36_b2_$b.json'));print('batch', $b, d['ms_per_step'], d['outputs_ok'])"; done
