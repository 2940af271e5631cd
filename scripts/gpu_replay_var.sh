set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_control.py tests/test_gpu_replay_warp.py tests/test_gpu_edge.py tests/test_gpu_random.py tests/test_decisions.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_replay.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_replay.log
for mb in 6; do
PALS_REPLAY_MINB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --queries 1000 --cfg3-queries 1000 --cfg5-traces 0 --sim-seeds 0 --predictions 1048576 --clusters 10000 --no-cpu-baseline > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err
done
