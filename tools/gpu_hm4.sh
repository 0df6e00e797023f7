#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/hm4.log
timeout 200 python tools/hm_bench.py >> gpurun_out/hm4.log 2>&1
for v in dqw8 dbg1 dbg2 dbg3; do
  FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_$v.so timeout 200 python tools/hm_bench.py >> gpurun_out/hm4.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_moe64_hm2 -f python tools/prof_moe.py --experts 64 --me 64 --iters 2 > gpurun_out/ncu_moe.log 2>&1
