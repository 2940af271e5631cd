# One GPU call: parity tests, smoke, the default bench + reference arm, the ncu launch list
# of the bench command and ncu --set full captures of the top kernels at the bench's sizes.
# Outputs land in gpurun_out/; scripts/refresh_profiles.sh <round> copies them to profiles/.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
START=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - START ))s" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
NCU="ncu --set full --clock-control none --import-source on -f"
# the launch list of the bench command itself (cold-cache, serialised: shares, not absolutes)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --sim-no-stream > gpurun_out/b_ncu.log 2>&1
# the select graph at cfg2's bench size (1e4 queries, 65,536 configs); launch 4 = a warm step
for k in k_scan k_eval_analytic k_sort_chunks k_merge_round k_assign_qprep k_finalize; do
  timeout 600 $NCU -k "regex:^$k" -s 3 -c 1 -o gpurun_out/prof_$k python scripts/select_quick.py cfg2 2 x > gpurun_out/ncu_$k.log 2>&1
done
# the replay at its bench size (1e6 traces x 3600 steps), thread layout
timeout 900 $NCU -k "regex:^k_replay$" -s 0 -c 1 -o gpurun_out/prof_k_replay python scripts/replay_quick.py 1000000 3600 > gpurun_out/ncu_k_replay.log 2>&1
timeout 900 $NCU -k "regex:k_allocate" -c 1 -o gpurun_out/prof_k_allocate python scripts/leg.py alloc > gpurun_out/ncu_k_allocate.log 2>&1
timeout 900 $NCU -k "regex:k_forest_eval_aos" -c 1 -o gpurun_out/prof_k_forest_eval_aos python scripts/leg.py forest > gpurun_out/ncu_k_forest.log 2>&1
timeout 900 $NCU -k "regex:k_front_scan" -c 1 -o gpurun_out/prof_k_front_scan python scripts/leg.py frontier > gpurun_out/ncu_k_front.log 2>&1
timeout 900 $NCU -k "regex:k_sim" -c 1 -o gpurun_out/prof_k_sim python scripts/leg.py sim > gpurun_out/ncu_k_sim.log 2>&1
ls -la gpurun_out
