set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_alloc.py -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_alloc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_alloc.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_alloc.json 2> gpurun_out/bench_alloc.err
echo "bench rc=$?" >> gpurun_out/bench_alloc.err
