#!/bin/bash
# A6 iteration batch: GPU tests, then MoE / prefill / paper micro-benchmark for the default library
# and every diagnostic variant under paper_2308_09723_b200/_variants/.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
run() {
  timeout 200 python tools/moe_bench.py 2>&1 | grep "decode_tc=0"
  timeout 200 python tools/tc_bench.py 2>&1
  timeout 400 python tools/paper_microbench.py --bits 4 --group 64 --rows 1 16 32 64 128 256 512 2048 2>&1 | grep geomean
}
echo "== default" > gpurun_out/ab.log; run >> gpurun_out/ab.log
for v in paper_2308_09723_b200/_variants/*.so; do
  [ -e "$v" ] || continue
  echo "== $v" >> gpurun_out/ab.log; FQ_LIB_PATH=$PWD/$v run >> gpurun_out/ab.log
done
