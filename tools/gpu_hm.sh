#!/bin/bash
# A6 two-half tiles: GPU tests, then mid-M timings with one- and two-half tiles.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo "pytest $?" >> gpurun_out/t.log
for hm in 1 default 2; do
  if [ $hm = default ]; then timeout 300 python tools/tc_mid.py > gpurun_out/hm_$hm.log 2>&1
  else FQ_TC_HM=$hm timeout 300 python tools/tc_mid.py > gpurun_out/hm_$hm.log 2>&1; fi
done
