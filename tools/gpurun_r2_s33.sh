#!/bin/bash
# Fused pass: results out by one bulk store (un-swizzled in place by the last DIT round).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "known_answers or tma_tile or pass_engine or lean or radix3 or squaring or convolution" > gpurun_out/s33_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s33_quick.log
tail -3 gpurun_out/s33_quick.log
grep -q "rc=0" gpurun_out/s33_quick.log || exit 1
for c in 3 33; do timeout 600 python tools/abtime.py --config $c --rounds 3 ablibs/lib_base.so ablibs/lib_obulk.so > gpurun_out/s33_ab_c$c.txt 2>&1; done
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_base.so ablibs/lib_obulk.so > gpurun_out/s33_ab_c4.txt 2>&1
timeout 900 python tools/abtime.py --config 5 --rounds 2 --steps 2 ablibs/lib_base.so ablibs/lib_obulk.so > gpurun_out/s33_ab_c5.txt 2>&1
grep "==" gpurun_out/s33_ab_c*.txt | cut -c1-300
