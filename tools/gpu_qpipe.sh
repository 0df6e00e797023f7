#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/qpipe.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for r in 1 2; do
FQ_QUANT_PIPE=0 timeout 200 python tools/quant_bench.py 2>&1 | sed 's/^/pipe0 /' >> gpurun_out/qpipe.log
timeout 200 python tools/quant_bench.py 2>&1 | sed 's/^/pipe1 /' >> gpurun_out/qpipe.log
done
