#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/v32.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
timeout 200 python tools/v32_bench.py >> gpurun_out/v32.log 2>&1
FQ_GEMM_PATH=tc FQ_TC_HM=1 timeout 200 python tools/v32_bench.py >> gpurun_out/v32.log 2>&1
FQ_GEMM_PATH=tc FQ_TC_HM=2 timeout 200 python tools/v32_bench.py >> gpurun_out/v32.log 2>&1
FQ_GEMM_PATH=tc FQ_TC_HM=2 FQ_TC_NO32=1 timeout 200 python tools/v32_bench.py >> gpurun_out/v32.log 2>&1
