#!/bin/bash
# ncu --set full of the decode kernel at M=1 (FC1), normal and skeleton (FQ_DEC_DEBUG=3) variants.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in 0 3; do
  FQ_DEC_DEBUG=$d timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m1_dbg$d -f python tools/prof_gemm.py --M ${PM:-1} --iters 3 > gpurun_out/ncu_dbg$d.log 2>&1
done
