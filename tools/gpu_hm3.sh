#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
timeout 300 python tools/tc_mid.py > gpurun_out/hm_rule.log 2>&1
timeout 400 python tools/paper_microbench.py --bits 4 --group 64 --rows 1 16 32 48 64 128 256 > gpurun_out/micro_hm.log 2>&1
