# parity suite + bench (replay legs at full size)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="--steps 10 --warmup 3 --predictions 1048576 --cfg3-queries 100000 --sim-seeds 0 --no-cpu-baseline"
timeout 900 python bench.py $B > gpurun_out/bench.json 2> gpurun_out/bench.err
