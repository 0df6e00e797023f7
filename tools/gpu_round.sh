#!/bin/bash
# Round-end evidence batch: tests, smoke, bench (with extras + cpu baseline), reference arm,
# ncu launch list of the bench command and full captures of the decode (M=1, M=16) and prefill kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m1 -f python tools/prof_gemm.py --M 1 --iters 3 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/dec_m16 -f python tools/prof_gemm.py --M 16 --iters 3 > gpurun_out/ncu16.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 -o gpurun_out/tc_m2048 -f python tools/prof_gemm.py --M 2048 --iters 2 > gpurun_out/ncutc.log 2>&1
