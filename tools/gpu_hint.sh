#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/hint.log
for r in 1 2; do
timeout 200 python tools/v32_bench.py >> gpurun_out/hint.log 2>&1
timeout 200 python tools/hm_bench.py >> gpurun_out/hint.log 2>&1
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_nohint.so timeout 200 python tools/v32_bench.py 2>&1 | sed 's/^/nohint /' >> gpurun_out/hint.log
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_nohint.so timeout 200 python tools/hm_bench.py >> gpurun_out/hint.log 2>&1
done
