#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m1 -f python tools/prof_gemm.py --M 1 --iters 3 > gpurun_out/ncu1.log 2>&1
