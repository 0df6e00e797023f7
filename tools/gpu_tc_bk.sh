# A6 stage-K A/B (FQ_TC_BK) + GPU tests; outputs under gpurun_out/
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/all_gpu.log 2>&1
for bk in 64 128; do FQ_TC_BK=$bk timeout 400 python tools/tc_mid.py >> gpurun_out/tc_bk.log 2>&1; done
