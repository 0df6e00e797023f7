#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/persist.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for r in 1 2; do
  FQ_DEC_PERSIST=0 timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/P0 /' >> gpurun_out/persist.log
  timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/P1 /' >> gpurun_out/persist.log
  FQ_GEMV_SPLITS=6 timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/P1S6 /' >> gpurun_out/persist.log
done
FQ_DEC_PERSIST=0 timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_p0.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_p1.log 2>&1
