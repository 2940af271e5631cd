set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/ab_prep.py > gpurun_out/ab_prep.log 2>&1
for m in 0 1; do
PALS_MERGE=$m timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_gpu_edge.py tests/test_gpu_random.py tests/test_gpu_pareto.py tests/test_forest.py -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_merge$m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_merge$m.log
done
