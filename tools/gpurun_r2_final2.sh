#!/bin/bash
# Round-2 evidence on one GPU box: all GPU tests, smoke, bench lines of every config (and the
# reference arm), launch lists, and ncu --set full captures exported as CSV (the .ncu-rep files
# stay on the box: they exceed the copy-back cap).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/ncu; rm -f /tmp/ncu/f2_*.ncu-rep
part=${1:-a}
if [ "$part" = a ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout=600 > gpurun_out/f2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f2_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f2_smoke.log
  timeout 600 python bench.py > gpurun_out/f2_b4.json 2> gpurun_out/f2_b4.err
  for c in 2 1 3 33 5; do timeout 900 python bench.py --config $c > gpurun_out/f2_b$c.json 2>gpurun_out/f2_b$c.err; done
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f2_bref4.json 2>gpurun_out/f2_bref4.err
  timeout 900 python bench.py --impl reference --config 2 --steps 3 --warmup 3 > gpurun_out/f2_bref2.json 2>gpurun_out/f2_bref2.err
  for c in 1 2 3 4 5; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches_cfg$c.csv python tools/profile_case.py --config $c --reps 2 > /dev/null 2>&1; done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_bench_launches_cfg4.csv python bench.py --steps 2 --warmup 3 > gpurun_out/f2_bench_under_ncu.log 2>&1
else
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_pack|k_pass|k_carry" -c 12 -o /tmp/ncu/f2_cfg4 python tools/profile_case.py --config 4 --reps 1 > gpurun_out/f2_ncu4.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -c 1 -o /tmp/ncu/f2_cfg2 python tools/profile_case.py --config 2 --reps 1 > gpurun_out/f2_ncu2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_pack|k_pass|k_carry" -c 6 -o /tmp/ncu/f2_cfg1 python tools/profile_case.py --config 1 --reps 1 > gpurun_out/f2_ncu1.log 2>&1
  for r in f2_cfg4 f2_cfg2 f2_cfg1; do
    ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
    ncu -i /tmp/ncu/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_source.csv 2>/dev/null
  done
  gzip -f gpurun_out/f2_*_source.csv
fi
ls -la gpurun_out | grep f2_ | head -60
