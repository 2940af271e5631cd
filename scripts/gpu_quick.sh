# parity tests + bench (+ replay register/occupancy variants) + launch list
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for mb in 6 8; do PALS_REPLAY_MINB=$mb timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_minb$mb.json 2>> gpurun_out/bench.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --traces 100000 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
