#!/bin/bash
# tools/mkvariant.sh NAME [extra nvcc flags...]: a self-contained copy of the package + bench under
# variants/NAME with libusk.so built with the given flags (tuning A/B runs on the GPU box).
set -e
cd "$(dirname "$0")/.."
N=$1; shift
D=variants/$N
rm -rf "$D"; mkdir -p "$D"
cp -r bench.py synth oracle include tools "$D"/
mkdir -p "$D/paper_2506_17255_b200"
cp -r paper_2506_17255_b200/*.py paper_2506_17255_b200/csrc "$D/paper_2506_17255_b200/"
[ -n "$VARIANT_QUERY" ] && cp "$VARIANT_QUERY" "$D/paper_2506_17255_b200/csrc/query.cu"
[ -n "$VARIANT_BUILD" ] && cp "$VARIANT_BUILD" "$D/paper_2506_17255_b200/csrc/build.cu"
cp oracle/liboracle.so "$D/oracle/" 2>/dev/null || true
USK_NVCC_FLAGS="$*" python "$D/paper_2506_17255_b200/build.py" > "$D/build.log" 2>&1 || { tail -20 "$D/build.log"; exit 1; }
rm -rf "$D/paper_2506_17255_b200/build"
echo "$D ready"
