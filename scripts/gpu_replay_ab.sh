# replay change: replay parity suite + the bench's replay legs
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_control.py tests/test_decisions.py tests/test_gpu_replay_warp.py tests/test_gpu_adapter.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r.log
B="--steps 5 --warmup 3 --predictions 1048576 --cfg3-queries 10000 --sim-seeds 0 --cfg5-traces 0 --no-cpu-baseline"
timeout 600 python bench.py $B > gpurun_out/bench_r.json 2> gpurun_out/bench_r.err
