set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SMALL="--steps 3 --warmup 1 --traces 20000 --trace-steps 360 --predictions 1048576 --no-cpu-baseline"
for c in 2048 4096; do for g in 1 2 4; do
PALS_CROSS_G=$g PALS_SORT_CHUNK=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_$g.csv python bench.py $SMALL > /dev/null 2>&1
done; done
PALS_CROSS_WALK=0 PALS_SORT_CHUNK=2048 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_2048_old.csv python bench.py $SMALL > /dev/null 2>&1
