#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/lazy2.log
for r in 1 2; do
timeout 200 python tools/v32_bench.py 2>&1 | grep "M=16\|M_e=16" | sed 's/^/dflt /' >> gpurun_out/lazy2.log
for v in lazy2 lazy2r96 lazy2r112; do
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_$v.so timeout 200 python tools/v32_bench.py 2>&1 | grep "M=16\|M_e=16" | sed "s/^/$v /" >> gpurun_out/lazy2.log
done; done
FQ_LIB_PATH=$PWD/paper_2308_09723_b200/_variants/libfq_lazy2.so timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x -k "tiny or dtypes or split_k_paths or multi_tile or full_size" > gpurun_out/tlazy.log 2>&1; echo "pytest $?" >> gpurun_out/tlazy.log
