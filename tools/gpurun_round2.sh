set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/t_parity.log
timeout 600 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
echo "bench rc=$?" >> gpurun_out/bench4.err
timeout 600 python bench.py --config 2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 3 > gpurun_out/ncu4.log 2>&1
echo done
