# parity suite + the 2-rank gloo bench path (shares cuda:0)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
PALS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus 2 --steps 3 --warmup 1 --traces 50000 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 200000 > gpurun_out/bench_2rank_gloo$i.json 2> gpurun_out/bench_2rank$i.err; echo "rc=$?" >> gpurun_out/bench_2rank$i.err
done
