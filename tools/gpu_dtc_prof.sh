#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
PM=1,16 DBGS=0,63 FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_prof.so timeout 300 python tools/dtc_prof.py > gpurun_out/dtcp.log 2>&1
