cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/hmdbg.log
for hm in 1 2; do for s in 1 2 8; do
  FQ_TC_HM=$hm FQ_TC_SPLITS=$s timeout 120 python tools/hm_dbg.py 32 4096 512 4 128 >> gpurun_out/hmdbg.log 2>&1
done; done
FQ_TC_HM=2 timeout 120 python tools/hm_dbg.py 64 1024 384 4 128 >> gpurun_out/hmdbg.log 2>&1
FQ_TC_HM=2 FQ_TC_SPLITS=1 timeout 120 python tools/hm_dbg.py 64 1024 384 4 128 >> gpurun_out/hmdbg.log 2>&1
