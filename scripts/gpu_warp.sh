set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_replay_warp.py tests/test_gpu_control.py -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_warp.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_warp.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --cfg5-traces 0 --cfg3-queries 100000 > gpurun_out/bench_warp.json 2> gpurun_out/bench_warp.err; echo "bench rc=$?" >> gpurun_out/bench_warp.err
