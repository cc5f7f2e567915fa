#!/bin/bash
# Single large pageable product: overlapped stages vs the locked path; sharded bench path at one rank.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
DECMUL_OVERLAP=1 timeout 300 tools/decmul bench mul --digits 100000000 --iters 10
DECMUL_OVERLAP=0 timeout 300 tools/decmul bench mul --digits 100000000 --iters 10
done
DECMUL_OVERLAP=1 timeout 300 tools/decmul bench mul --digits 30000000 --iters 10
DECMUL_OVERLAP=0 timeout 300 tools/decmul bench mul --digits 30000000 --iters 10
timeout 900 python bench.py --config 4 --sharded --steps 5 > gpurun_out/s20_b4_sharded.json 2> gpurun_out/s20_b4_sharded.err; python -c "
import json;d=json.load(open('gpurun_out/s20_b4_sharded.json'));print(d['ms_per_step'], d.get('outputs_ok'), d['e2e'])" || tail -5 gpurun_out/s20_b4_sharded.err
