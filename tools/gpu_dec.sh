#!/bin/bash
# Decode-kernel iteration batch: parity tests, then the M sweep for the default library and for
# every diagnostic variant under paper_2308_09723_b200/_variants/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_moe.py tests/test_gpu_tp.py -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
echo "== default" > gpurun_out/sweep.log
timeout 300 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1
for v in paper_2308_09723_b200/_variants/*.so; do
  [ -e "$v" ] || continue
  echo "== $v" >> gpurun_out/sweep.log
  FQ_LIB_PATH=$PWD/$v timeout 300 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1
done
if [ -n "${DTC}" ]; then
  echo "== default FQ_DECODE_TC=1" >> gpurun_out/sweep.log
  FQ_DECODE_TC=1 timeout 300 python tools/dec_sweep.py ${SWEEP_ARGS} >> gpurun_out/sweep.log 2>&1
fi
