#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 17 24 32 > gpurun_out/micro_r_dec.log 2>&1
FQ_GEMM_PATH=tc timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 17 24 32 > gpurun_out/micro_r_tc.log 2>&1
FQ_GEMM_PATH=tc timeout 200 python tools/v32_bench.py > gpurun_out/route_tc.log 2>&1
