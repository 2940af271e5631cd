# parity tests + bench (+ replay register/occupancy variants) + launch list
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for mb in 6 8; do PALS_REPLAY_MINB=$mb timeout 600 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_minb$mb.json 2>> gpurun_out/bench.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --traces 100000 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
# the N>1 code path on one GPU: two ranks with gloo collectives sharing cuda:0
PALS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 1 --traces 50000 --predictions 1048576 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank.err; echo "rc=$?" >> gpurun_out/bench_2rank.err
