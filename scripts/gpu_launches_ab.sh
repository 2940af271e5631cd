set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SMALL="--steps 3 --warmup 1 --traces 20000 --trace-steps 360 --predictions 1048576 --no-cpu-baseline"
for c in 4096 2048; do
PALS_SORT_CHUNK=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py $SMALL > /dev/null 2>&1
done
