#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
timeout 200 python tools/v32_bench.py > gpurun_out/route.log 2>&1
timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 1 16 32 64 > gpurun_out/micro_route.log 2>&1
