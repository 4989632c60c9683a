#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Compiles the *unmodified* reference library from its
# sources where they lie under /root/reference (never copied into this repo),
# plus oracle/ref_shim.cpp, into oracle/_ref/librespar_ref.so.  The reference's
# own CMake build is not used (its vendored json/doctest/CLI11 are absent);
# nlohmann/json 3.11.3 comes from the cudnn_frontend headers in the venv
# (SURVEY.md §8c).  Output goes only to oracle/_ref/ (git-ignored, but it travels
# to the GPU box with gpurun so bench.py --impl reference can run there).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${RESPAR_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference sources not found at $REF (skipping; prebuilt oracle/_ref is used)" >&2
  exit 0
fi
JSON_DIR="$(python - <<'EOF'
import os, site, sys
for p in site.getsitepackages():
    d = os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann")
    if os.path.isfile(os.path.join(d, "json.hpp")):
        print(d); sys.exit(0)
sys.exit(1)
EOF
)"
mkdir -p "$OUT"
SRCS=(tensor network penalty decoupled runtime config dataset metrics experiment gradcheck)
FILES=()
for s in "${SRCS[@]}"; do FILES+=("$REF/src/$s.cpp"); done
g++ -std=c++20 -O2 -fPIC -shared -pthread \
    -I"$REF/include" -isystem "$JSON_DIR" \
    "${FILES[@]}" "$HERE/ref_shim.cpp" \
    -o "$OUT/librespar_ref.so.tmp"
mv "$OUT/librespar_ref.so.tmp" "$OUT/librespar_ref.so"
echo "build_ref: wrote $OUT/librespar_ref.so"
