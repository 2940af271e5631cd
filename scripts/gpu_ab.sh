# A/B of the sort/cross variants: parity tests per variant + bench + launch list
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1024 2048; do
  PALS_SORT_CHUNK=$c timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_edge.py tests/test_forest.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_chunk$c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_chunk$c.log
done
for c in 4096 2048 1024; do
  PALS_SORT_CHUNK=$c timeout 600 python bench.py --no-cpu-baseline --steps 10 --traces 200000 --predictions 1048576 > gpurun_out/bench_chunk$c.json 2>> gpurun_out/bench.err
done
SMALL="--steps 3 --warmup 1 --traces 20000 --trace-steps 360 --predictions 1048576 --no-cpu-baseline"
for c in 1024 2048; do
PALS_SORT_CHUNK=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py $SMALL > /dev/null 2>&1
done
