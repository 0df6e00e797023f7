#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_fc2_m64_dqg2 -f python tools/prof_gemm.py --M 64 --K 49152 --N 12288 --iters 2 > gpurun_out/ncu_a6a.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_fc1_m64 -f python tools/prof_gemm.py --M 64 --iters 2 > gpurun_out/ncu_a6b.log 2>&1
