#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_m2048 -f python tools/prof_gemm.py --M 2048 --iters 2 > gpurun_out/ncu_tc.log 2>&1
