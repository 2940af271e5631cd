# ncu --set full of the rank kernels of the cfg2 step (cluster path and chunk sort)
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SMALL="--steps 1 --warmup 1 --traces 2000 --trace-steps 60 --predictions 1048576 --cfg3-queries 10000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rank_cluster -s 8 -c 1 -o gpurun_out/prof_k_rank_cluster python bench.py $SMALL > gpurun_out/ncu_rc.log 2>&1
PALS_RANK_CLUSTER=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sort_chunks|k_merge_round" -s 14 -c 2 -o gpurun_out/prof_k_sort python bench.py $SMALL > gpurun_out/ncu_sort.log 2>&1
