# A/B of select-step variants on the captured cfg2 step (PDL edges on, no scan events)
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-base}; do echo "== $v"; PALS_GPU_LIB=_variants/$v.so timeout 300 python scripts/select_quick.py cfg2 200 x graph 2>&1 | tail -1; done
