set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="--steps 3 --warmup 1 --traces 50000 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 100000 --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/repro1.json 2> gpurun_out/repro1.err; echo "rc=$?" >> gpurun_out/repro1.err
timeout 600 compute-sanitizer --print-limit 5 python bench.py $A > gpurun_out/repro_san.json 2> gpurun_out/repro_san.err; echo "rc=$?" >> gpurun_out/repro_san.err
