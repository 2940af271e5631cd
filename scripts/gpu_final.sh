# Round-end evidence: parity suite, smoke, default bench + reference arm, the 2-rank gloo
# path of bench.py (N>1 code incl. the cfg5 strong shard + gather), launch list, and
# ncu --set full captures of the top kernels.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
START=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
PALS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --traces 50000 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 200000 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank.err; echo "rc=$?" >> gpurun_out/bench_2rank.err
SMALL="--steps 2 --warmup 1 --traces 100000 --predictions 4194304 --cfg3-queries 100000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $SMALL > gpurun_out/b_ncu.log 2>&1
for k in "k_scan\\(" "k_sort_chunks<\\(int\\)512, \\(int\\)4>" "k_merge_round<\\(int\\)512, \\(int\\)2>" k_forest_eval_aos k_assign_qprep k_allocate k_front_scan k_finalize; do
  n=${k%%[<\\]*}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 2 -c 1 -o gpurun_out/prof_$n python bench.py $SMALL > gpurun_out/ncu_$n.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_k_replay python bench.py --steps 1 --warmup 1 --trace-steps 300 --predictions 1048576 --cfg3-queries 100000 --cfg5-traces 0 --sim-seeds 0 --no-cpu-baseline > gpurun_out/ncu_k_replay.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sim -s 1 -c 1 -o gpurun_out/prof_k_sim python scripts/sim_quick.py 16 > gpurun_out/ncu_k_sim.log 2>&1
ls -la gpurun_out
