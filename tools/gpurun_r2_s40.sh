#!/bin/bash
# Row passes: the butterfly table by a bulk copy on the tile's barrier (configs 3, 4).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 -k "known_answers or tma_tile or pass_engine or lean or radix3" > gpurun_out/s40_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s40_quick.log
tail -3 gpurun_out/s40_quick.log
grep -q "rc=0" gpurun_out/s40_quick.log || exit 1
timeout 600 python tools/abtime.py --config 3 --rounds 3 ablibs/lib_base.so ablibs/lib_tbl.so > gpurun_out/s40_ab_c3.txt 2>&1
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_base.so ablibs/lib_tbl.so > gpurun_out/s40_ab_c4.txt 2>&1
grep "==" gpurun_out/s40_ab_c*.txt | cut -c1-300
