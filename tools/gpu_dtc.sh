#!/bin/bash
# tcgen05 decode iteration batch: decode parity tests, then the M sweep (tcgen05 and mma.sync).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_moe.py -m gpu -q -x ${PYTEST_K} > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
echo "== default (mma.sync stream-K)" > gpurun_out/sweep.log
timeout 200 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1
echo "== mma.sync split-K grid" >> gpurun_out/sweep.log
FQ_GEMV_SK=0 timeout 200 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1


for v in paper_2308_09723_b200/_variants/*.so; do
  [ -e "$v" ] || continue
  echo "== $v" >> gpurun_out/sweep.log
  FQ_LIB_PATH=$PWD/$v timeout 100 python tools/dec_sweep.py --M 9 16 >> gpurun_out/sweep.log 2>&1
done
