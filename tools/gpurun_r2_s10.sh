#!/bin/bash
# PCIe duplex probe, stage trace of overlapped config-4 products, TMA store epilogue A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/pcie_duplex.py > gpurun_out/s10_pcie.txt 2>&1; cat gpurun_out/s10_pcie.txt
DECMUL_OVERLAP_TRACE=1 timeout 600 python bench.py --steps 8 > gpurun_out/s10_b4.json 2> gpurun_out/s10_b4_trace.txt
grep overlap gpurun_out/s10_b4_trace.txt | tail -12
timeout 900 python tools/abtime.py --config 4 --rounds 3 --steps 5 ablibs/lib_tma.so ablibs/lib_tmast.so > gpurun_out/s10_ab_c4.txt 2>&1
timeout 600 python tools/abtime.py --config 3 --rounds 3 ablibs/lib_tma.so ablibs/lib_tmast.so > gpurun_out/s10_ab_c3.txt 2>&1
timeout 900 python tools/abtime.py --config 5 --rounds 2 --steps 2 ablibs/lib_tma.so ablibs/lib_tmast.so > gpurun_out/s10_ab_c5.txt 2>&1
grep "==" gpurun_out/s10_ab_c*.txt | cut -c1-330
