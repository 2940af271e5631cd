set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SMALL="--steps 2 --warmup 1 --traces 100000 --predictions 4194304 --cfg3-queries 100000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
for k in "k_sort_chunks<\\(int\\)512, \\(int\\)4>" "k_merge_round<\\(int\\)512, \\(int\\)2>"; do
  n=${k%%[<\\]*}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 2 -c 1 -o gpurun_out/prof_$n python bench.py $SMALL > gpurun_out/ncu_$n.log 2>&1
done
