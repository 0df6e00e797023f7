#!/bin/bash
mkdir -p gpurun_out
FQ_DECODE_TC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_tc_kernel -s 2 -c 1 -o gpurun_out/dtc_m1 -f python tools/prof_gemm.py --M 1 --iters 3 > gpurun_out/ncu_dtc.log 2>&1
