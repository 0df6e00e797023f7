mkdir -p gpurun_out
timeout 300 python tools/tc_mid.py quick > gpurun_out/tc_dbg.log 2>&1
for v in dbg3 dbg1 dbg2; do FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_$v.so timeout 300 python tools/tc_mid.py quick >> gpurun_out/tc_dbg.log 2>&1; done
