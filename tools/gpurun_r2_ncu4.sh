#!/bin/bash
# ncu --set full of the config-4 chain (one launch of each kernel kind) and k_small (config 2);
# raw-page CSV + source-page CSV exported on the box (the .ncu-rep files exceed the copy-back cap).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/ncu
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_pack_radix3|k_pass_fwd|k_pass_fused|k_pass_inv|k_carry" -c 9 -o /tmp/ncu/r02_cfg4 python tools/profile_case.py --config 4 --reps 1 > gpurun_out/ncu_cfg4.log 2>&1
echo rc=$? >> gpurun_out/ncu_cfg4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -o /tmp/ncu/r02_k_small python tools/profile_case.py --config 2 --reps 1 > gpurun_out/ncu_cfg2.log 2>&1
for r in r02_cfg4 r02_k_small; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_source.csv 2>/dev/null
done
gzip -f gpurun_out/*_source.csv
ls -la gpurun_out
