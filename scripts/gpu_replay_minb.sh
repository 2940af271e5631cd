# replay occupancy A/B (launch bounds 6 vs 8 CTAs/SM) on the bench's replay legs
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--steps 5 --warmup 3 --predictions 1048576 --cfg3-queries 10000 --sim-seeds 0 --cfg5-traces 0 --no-cpu-baseline"
for m in 6 8 1; do
PALS_REPLAY_MINB=$m timeout 600 python bench.py $B > gpurun_out/bench_minb$m.json 2> gpurun_out/bench_minb$m.err
done
