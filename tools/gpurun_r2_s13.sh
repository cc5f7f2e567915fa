#!/bin/bash
# Mixed concurrent traffic test, then the final ncu --set full captures (part b of gpurun_r2_final2.sh).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=600 -k "mixed_concurrent or concurrent_large" > gpurun_out/s13_quick.log 2>&1; echo "rc=$?" >> gpurun_out/s13_quick.log
tail -4 gpurun_out/s13_quick.log
bash tools/gpurun_r2_final2.sh b
