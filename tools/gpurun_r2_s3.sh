#!/bin/bash
# Round-2 re-entry check on one GPU box: GPU tests, smoke, the default (config 4) bench line and
# config 2, then ncu --set full of the config-4 chain and k_small, exported as raw/source CSV.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/s3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s3_smoke.log
timeout 600 python bench.py > gpurun_out/s3_b4.json 2> gpurun_out/s3_b4.err
timeout 600 python bench.py --config 2 > gpurun_out/s3_b2.json 2> gpurun_out/s3_b2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_pack|k_pass|k_carry" -c 9 -o /tmp/ncu/s3_cfg4 python tools/profile_case.py --config 4 --reps 1 > gpurun_out/s3_ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -o /tmp/ncu/s3_cfg2 python tools/profile_case.py --config 2 --reps 1 > gpurun_out/s3_ncu2.log 2>&1
for r in s3_cfg4 s3_cfg2; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_source.csv 2>/dev/null
done
gzip -f gpurun_out/s3_*_source.csv
ls -la gpurun_out | grep s3_
