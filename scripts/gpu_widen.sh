set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_alloc.py tests/test_gpu_pareto.py tests/test_gpu_adapter.py -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_widen.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_widen.log
./tests/cpp/test_adapter . > gpurun_out/adapter.log 2>&1; echo "adapter rc=$?" >> gpurun_out/adapter.log
