# One GPU call: parity tests, the default bench, the ncu launch list and two
# ncu --set full captures (k_scan, k_replay). Outputs land in gpurun_out/.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --traces 100000 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_scan python bench.py --steps 2 --warmup 1 --traces 20000 --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_replay python bench.py --steps 1 --warmup 1 --traces 100000 --trace-steps 600 --no-cpu-baseline > gpurun_out/ncu_replay.log 2>&1
ls -la gpurun_out
