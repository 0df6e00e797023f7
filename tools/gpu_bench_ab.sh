cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_pdl.log 2>&1
FQ_PDL=0 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_nopdl.log 2>&1
