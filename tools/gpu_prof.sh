#!/bin/bash
# ncu captures of the decode kernel (FC1 M=1 and M=16, int4) + quantizer.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m1 -f python tools/prof_gemm.py --M 1 --iters 3 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m16 -f python tools/prof_gemm.py --M 16 --iters 3 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:quantize_kernel -s 1 -c 1 -o gpurun_out/quant -f python tools/prof_gemm.py --M 1 --iters 2 --quantize > gpurun_out/ncu3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1
