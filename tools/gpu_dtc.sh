#!/bin/bash
# tcgen05 decode diagnostics: FQ_DTC_DBG sweep for the default library and each variant.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
echo "== default" > gpurun_out/dtcd.log
timeout 300 python tools/dtc_dbg.py >> gpurun_out/dtcd.log 2>&1
for v in paper_2308_09723_b200/_variants/*.so; do
  [ -e "$v" ] || continue
  echo "== $v" >> gpurun_out/dtcd.log
  FQ_LIB_PATH=$PWD/$v timeout 300 python tools/dtc_dbg.py >> gpurun_out/dtcd.log 2>&1
done
if [ -n "${NCU}" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_tc -s 2 -c 1 -o gpurun_out/dtc_m1 -f python tools/prof_gemm.py --M 1 --iters 3 > gpurun_out/ncu_dtc.log 2>&1
fi
