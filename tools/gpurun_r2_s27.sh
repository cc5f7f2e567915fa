#!/bin/bash
# Chunk count of the batch pipeline under overlapped calls (config 2, three threads).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 1 2 3 5 9; do DECMUL_PIPE_CHUNKS=$k timeout 300 python bench.py --config 2 --e2e-threads 3 > gpurun_out/s27_k$k.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/s27_k$k.json'));print('chunks', $k, 'threads 3', d['e2e']['ms_per_step'], 'single', d['e2e'].get('single_call_ms'))"; done
