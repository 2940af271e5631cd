# A/B of k_scan variants (_variants/*.so, scripts/build_variants.sh): cfg2 / cfg3 select step
# and scan timings, then the CTA phase trace of the trace builds.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-head cps3 cps4}; do
  for c in cfg2 cfg3; do
    r=30; [ $c = cfg3 ] && r=5
    echo "== $v $c"; PALS_GPU_LIB=_variants/$v.so timeout 300 python scripts/select_quick.py $c $r 2>&1 | tail -3
  done
done
for v in ${TRACES:-headtrace trace}; do
  echo "== trace $v"; PALS_GPU_LIB=_variants/$v.so timeout 300 python scripts/scan_trace.py cfg2 2>&1 | tail -20
  [ -f gpurun_out/scan_trace_cfg2.npy ] && mv gpurun_out/scan_trace_cfg2.npy gpurun_out/scan_trace_cfg2_$v.npy
done
