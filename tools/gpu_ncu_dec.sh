#!/bin/bash
# ncu --set full of fq::decode_kernel for each M in $PMS (FC1 int4 g128).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in ${PMS:-1 16}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m$m -f python tools/prof_gemm.py --M $m --iters 3 > gpurun_out/ncu_m$m.log 2>&1
done
