#!/bin/bash
# tcgen05 decode iteration batch: decode parity tests, then the M sweep (tcgen05 and mma.sync).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_moe.py -m gpu -q -x ${PYTEST_K} > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
echo "== tcgen05" > gpurun_out/sweep.log
timeout 200 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1
echo "== mma.sync" >> gpurun_out/sweep.log
FQ_DECODE_TC=0 timeout 200 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1


