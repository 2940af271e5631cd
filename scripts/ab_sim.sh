# A/B of k_sim variants (_variants/*.so): the queue-plant leg at the bench's seed count,
# streamed (whole call) and uploaded first (the kernel's own time)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-sbase}; do
  for f in "" --sim-no-stream; do
    echo "== $v $f"
    PALS_GPU_LIB=_variants/$v.so timeout 600 python scripts/sim_quick.py ${SEEDS:-256} $f 2>&1 |
      python -c "import json,sys; l=sys.stdin.read().strip().splitlines(); r=json.loads(l[-1]); print(r.get('value'), r.get('e2e', {}).get('value') if isinstance(r.get('e2e'), dict) else r.get('e2e'), r.get('ms_per_step'))" 2>&1 | tail -2
  done
done
