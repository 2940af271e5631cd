#!/usr/bin/env bash
# Build tests/cpp/test_adapter: the reference's headers (for the CPU side of the
# comparison and the reference types the adapter speaks) + include/wattserve_gpu.hpp
# linked against paper_2605_21427_b200/libpals_gpu.so. Needs /root/reference, so it
# is built in the build container; the binary travels to the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${REF_ROOT:-/root/reference/proj}"
JSON_INC="$(python3 -c "import site,os;print(next((os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages() if os.path.exists(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann/json.hpp'))),''))")"
if [ ! -d "$REF/include/wattserve" ]; then
  echo "reference headers absent: keeping prebuilt test_adapter (if any)"; exit 0
fi
g++ -std=c++20 -O2 -I"$REF/include" -I"$JSON_INC" -I"$ROOT/include" \
    "$HERE/test_adapter.cpp" -o "$HERE/test_adapter" \
    -L"$ROOT/paper_2605_21427_b200" -lpals_gpu -Wl,-rpath,'$ORIGIN/../../paper_2605_21427_b200'
echo "built $HERE/test_adapter"
