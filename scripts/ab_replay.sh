# A/B of k_replay variants (_variants/*.so): cfg4 thread / warp / caller-trace layouts,
# summary digest (the variants must agree byte for byte)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-rhead rnew}; do
  echo "== $v"; PALS_GPU_LIB=_variants/$v.so timeout 600 python scripts/replay_quick.py ${NT:-1000000} ${NS:-3600} 2>&1 | tail -2
done
