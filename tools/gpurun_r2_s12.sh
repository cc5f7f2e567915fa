#!/bin/bash
# A/B for small transforms: TMA on the 4-column tiles, mid-kernel PDL trigger (configs 1, 3; a
# 3e6 x 2e6-digit product through config 1's timing loop is covered by abtime --config 1 only).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1 3; do timeout 900 python tools/abtime.py --config $c --rounds 3 ablibs/lib_base.so ablibs/lib_narrow.so ablibs/lib_pdlmid.so ablibs/lib_pdlmid_narrow.so > gpurun_out/s12_ab_c$c.txt 2>&1; done
timeout 900 python tools/abtime.py --config 4 --rounds 2 --steps 5 ablibs/lib_base.so ablibs/lib_pdlmid.so > gpurun_out/s12_ab_c4.txt 2>&1
grep "==" gpurun_out/s12_ab_c*.txt | cut -c1-330
