# replay occupancy A/B (6 / 7 / 8 CTAs per SM) on the bench's replay legs + replay parity
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 7 8; do
PALS_REPLAY_MINB=$m timeout 900 python -m pytest tests/test_gpu_control.py tests/test_decisions.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_minb$m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_minb$m.log
done
B="--steps 5 --warmup 3 --predictions 1048576 --cfg3-queries 10000 --sim-seeds 0 --cfg5-traces 0 --no-cpu-baseline"
for m in 6 7 8; do
PALS_REPLAY_MINB=$m timeout 600 python bench.py $B > gpurun_out/bench_minb$m.json 2> gpurun_out/bench_minb$m.err
done
