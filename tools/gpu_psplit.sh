#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for r in 1 2; do
FQ_TC_SPLITS=1 timeout 300 python tools/tc_mid.py 2>&1 | grep "M=256\|M=2048" | sed 's/^/s1 /' >> gpurun_out/psplit.log
timeout 300 python tools/tc_mid.py 2>&1 | grep "M=256\|M=2048" | sed 's/^/plan /' >> gpurun_out/psplit.log
done
timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 256 512 2048 > gpurun_out/micro_psplit.log 2>&1
FQ_TC_SPLITS=1 timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 512 2048 > gpurun_out/micro_psplit_s1.log 2>&1
