#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
timeout 300 python tools/tc_mid.py > gpurun_out/dqg_rule.log 2>&1
