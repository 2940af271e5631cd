set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/ab_prep.py > gpurun_out/ab_prep.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
