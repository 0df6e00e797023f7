#!/bin/bash
# Round-end evidence batch: tests, smoke, bench (extras + cpu baseline), reference arm, launch list,
# decode / prefill ncu captures (gpu_round.sh), plus the paper micro-benchmark at 17..64 rows.
cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh
timeout 400 python tools/paper_microbench.py --bits 4 --group 128 --rows 1 8 16 24 32 48 64 > gpurun_out/micro_final.log 2>&1
