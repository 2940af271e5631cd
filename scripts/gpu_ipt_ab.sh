# chunk-size A/B of the block sort (2,048 vs 4,096 keys, 4 keys per thread): parity + cfg2 bench lines
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PALS_SORT_CHUNK=4096 timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_edge.py tests/test_gpu_random.py tests/test_gpu_pareto.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_ipt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ipt.log
B="--steps 10 --warmup 3 --traces 20000 --trace-steps 360 --predictions 1048576 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
for c in 2048 4096; do
PALS_SORT_CHUNK=$c timeout 600 python bench.py $B > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
