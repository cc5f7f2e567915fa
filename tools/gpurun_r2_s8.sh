#!/bin/bash
# TMA (cp.async.bulk.tensor.2d) staging of full-width row tiles vs the cp.async burst: quick
# parity first (a hang here must not eat the budget), then A/B on configs 3, 4, 5; full GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=120 -k "known_answers or forced_six or rho or convolution_hook" > gpurun_out/s8_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s8_quick.log
tail -3 gpurun_out/s8_quick.log
grep -q "rc=0" gpurun_out/s8_quick.log || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s8_tests.log
tail -3 gpurun_out/s8_tests.log
timeout 600 python tools/abtime.py --config 3 --rounds 3 ablibs/lib_cpasync.so ablibs/lib_tma.so > gpurun_out/s8_ab_c3.txt 2>&1
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_cpasync.so ablibs/lib_tma.so > gpurun_out/s8_ab_c4.txt 2>&1
timeout 900 python tools/abtime.py --config 5 --rounds 2 --steps 2 ablibs/lib_cpasync.so ablibs/lib_tma.so > gpurun_out/s8_ab_c5.txt 2>&1
grep "==" gpurun_out/s8_ab_c*.txt | cut -c1-330
