set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--gpus 2 --steps 3 --warmup 1 --traces 50000 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 200000 --no-cpu-baseline"
cat > /tmp/sanwrap.sh <<'EOW'
#!/bin/bash
exec compute-sanitizer --print-limit 3 --log-file /root/repo/gpurun_out/san_rank$RANK.log python bench.py "$@"
EOW
chmod +x /tmp/sanwrap.sh
PALS_BENCH_BACKEND=gloo CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 --no-python /tmp/sanwrap.sh $A > gpurun_out/r2.json 2> gpurun_out/r2.err; echo "rc=$?" >> gpurun_out/r2.err
