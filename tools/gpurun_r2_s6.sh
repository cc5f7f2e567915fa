#!/bin/bash
# A/B: fast constant-map carry paths and the prefix-map top-limb probe (configs 1, 2, 3, 4); GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s6_tests.log
tail -3 gpurun_out/s6_tests.log
for c in 1 2 3; do timeout 600 python tools/abtime.py --config $c --rounds 3 ablibs/lib_base.so ablibs/lib_mapslow.so ablibs/lib_mapfast.so > gpurun_out/s6_ab_c$c.txt 2>&1; done
timeout 900 python tools/abtime.py --config 4 --rounds 2 --steps 5 ablibs/lib_mapslow.so ablibs/lib_mapfast.so > gpurun_out/s6_ab_c4.txt 2>&1
grep "==" gpurun_out/s6_ab_c*.txt | cut -c1-330
