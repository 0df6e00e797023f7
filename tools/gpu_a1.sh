#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/a1.log
timeout 600 python -m pytest tests/test_gpu_quant.py tests/test_gpu_moe.py -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for r in 1 2; do
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_a1old.so timeout 200 python tools/quant_bench.py 2>&1 | grep adapt | sed 's/^/old /' >> gpurun_out/a1.log
timeout 200 python tools/quant_bench.py 2>&1 | grep adapt | sed 's/^/new /' >> gpurun_out/a1.log
done
