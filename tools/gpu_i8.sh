#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/i8.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for r in 1 2; do
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_oldi8.so timeout 300 python tools/tc_mid.py 2>&1 | grep int8 | sed 's/^/old /' >> gpurun_out/i8.log
timeout 300 python tools/tc_mid.py 2>&1 | grep int8 | sed 's/^/new /' >> gpurun_out/i8.log
done
