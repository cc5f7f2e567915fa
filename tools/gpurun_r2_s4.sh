#!/bin/bash
# A/B: per-group (merged radix-3) pass-1 table prefetch variants on config 4; ncu of the carry kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_base.so ablibs/lib_nopf.so ablibs/lib_ipf.so ablibs/lib_both.so > gpurun_out/s4_ab_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_carry" -c 3 -o /tmp/ncu/s4_carry4 python tools/profile_case.py --config 4 --reps 1 > gpurun_out/s4_ncu_carry4.log 2>&1
ncu -i /tmp/ncu/s4_carry4.ncu-rep --page raw --csv > gpurun_out/s4_carry4_raw.csv 2>/dev/null
ncu -i /tmp/ncu/s4_carry4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/s4_carry4_source.csv 2>/dev/null
gzip -f gpurun_out/s4_carry4_source.csv
grep "==" gpurun_out/s4_ab_c4.txt | cut -c1-300
