# default bench + the 2-rank gloo path (N>1 code incl. the cfg5 strong shard + gather)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
PALS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 1 --traces 50000 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 200000 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank.err; echo "rc=$?" >> gpurun_out/bench_2rank.err
