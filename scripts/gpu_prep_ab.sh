# parity suite, default-size bench line, launch list of the cfg2/cfg3 steps
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="--steps 10 --warmup 3 --traces 20000 --trace-steps 360 --predictions 1048576 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
timeout 600 python bench.py $B > gpurun_out/bench.json 2> gpurun_out/bench.err
SMALL="--steps 2 --warmup 1 --traces 20000 --trace-steps 60 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $SMALL > /dev/null 2>&1
