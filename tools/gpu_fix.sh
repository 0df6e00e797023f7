#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/fix.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
OLD=$PWD/paper_2308_09723_b200/_variants/libfq_oldfix.so
for r in 1 2; do
  FQ_LIB_PATH=$OLD timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/old /' >> gpurun_out/fix.log
  timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/new /' >> gpurun_out/fix.log
  FQ_LIB_PATH=$OLD timeout 200 python tools/hm_bench.py 2>&1 | sed 's/^/old /' >> gpurun_out/fix.log
  timeout 200 python tools/hm_bench.py 2>&1 | sed 's/^/new /' >> gpurun_out/fix.log
done
FQ_LIB_PATH=$OLD timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_old.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_new.log 2>&1
FQ_LIB_PATH=$OLD timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_old2.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_new2.log 2>&1
