#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/dqw16.log
V=$PWD/paper_2308_09723_b200/_variants/libfq_dqw16.so
FQ_LIB_PATH=$V timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x -k "tc or prefill or large_m" > gpurun_out/t16.log 2>&1; echo "pytest $?" >> gpurun_out/t16.log
for r in 1 2; do
timeout 300 python tools/tc_bench.py 2>&1 | sed 's/^/dflt /' >> gpurun_out/dqw16.log
FQ_LIB_PATH=$V timeout 300 python tools/tc_bench.py 2>&1 | sed 's/^/dqw16 /' >> gpurun_out/dqw16.log
done
