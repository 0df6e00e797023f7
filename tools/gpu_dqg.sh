#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
timeout 300 python tools/tc_mid.py > gpurun_out/dqg2.log 2>&1
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_dqg1.so timeout 300 python tools/tc_mid.py > gpurun_out/dqg1.log 2>&1
FQ_GEMM_PATH=tc FQ_TC_HM=2 timeout 200 python tools/v32_bench.py > gpurun_out/dqg2_v32.log 2>&1
timeout 400 python tools/paper_microbench.py --bits 4 --group 64 --rows 32 64 128 256 > gpurun_out/micro_dqg2.log 2>&1
