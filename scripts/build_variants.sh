#!/usr/bin/env bash
# Build kernel A/B variants of libpals_gpu.so: one source (SRC, default replay.cu) recompiled
# with each -D set, linked with the regular objects into _variants/<name>.so (select with
# PALS_GPU_LIB=...).
#   SRC=plan.cu scripts/build_variants.sh name1="-DX=1 -DY=1" name2="-DX=1" ...
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
B="$ROOT/paper_2605_21427_b200/_build"; C="$ROOT/paper_2605_21427_b200/csrc"; O="$ROOT/_variants"
mkdir -p "$O"
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --extended-lambda -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -O3"
SRC=${SRC:-replay.cu}
for kv in "$@"; do
  name="${kv%%=*}"; defs="${kv#*=}"
  ( $NV $FL $defs -c "$C/$SRC" -o "$O/$name.$SRC.o" &&
    objs=$(ls $B/*.o | grep -v "/$SRC.o") &&
    $NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$O/$name.so" $objs "$O/$name.$SRC.o" &&
    echo "built $O/$name.so" ) &
done
wait
