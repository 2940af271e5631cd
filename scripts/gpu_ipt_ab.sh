# block sort keys-per-thread A/B (8 vs 4): select parity + cfg2 bench line + launch list
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PALS_SORT_IPT=4 timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_edge.py tests/test_gpu_random.py tests/test_gpu_pareto.py -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_ipt4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ipt4.log
B="--steps 10 --warmup 3 --traces 20000 --trace-steps 360 --predictions 1048576 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
for i in 4 8; do
PALS_SORT_IPT=$i timeout 600 python bench.py $B > gpurun_out/bench_ipt$i.json 2> gpurun_out/bench_ipt$i.err
done
SMALL="--steps 2 --warmup 1 --traces 20000 --trace-steps 60 --predictions 1048576 --cfg3-queries 10000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
PALS_SORT_IPT=4 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ipt4.csv python bench.py $SMALL > /dev/null 2>&1
