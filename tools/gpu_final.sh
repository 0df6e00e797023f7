#!/bin/bash
# Round-end evidence batch (after the A6 two-half tiles): everything in gpu_round.sh, plus the MoE
# M_e = 32 route A/B (decode MT=4 vs A6 two-half tiles) and an ncu capture of A6 on OPT-175B FC2 M=64.
cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh
FQ_GEMM_PATH=tc timeout 200 python tools/hm_bench.py > gpurun_out/hm_tc_forced.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_fc2_m64 -f python tools/prof_gemm.py --M 64 --K 49152 --N 12288 --iters 2 > gpurun_out/ncutc2.log 2>&1
