#!/bin/bash
# Build libtide_b200.so from the csrc/ of a git revision (or the work tree) into
# tools/_libs/<name>.so, for A/B timing on one box: TIDE_PROBE_LIB=... tools/k1_probe.py
#   tools/build_variant.sh base HEAD     |   tools/build_variant.sh new work
set -e
NAME=$1; REV=${2:-work}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/paper_2603_21365_b200/csrc" "$TMP/include" "$ROOT/tools/_libs"
if [ "$REV" = work ]; then
  cp "$ROOT"/paper_2603_21365_b200/csrc/* "$TMP/paper_2603_21365_b200/csrc/"; cp "$ROOT"/include/* "$TMP/include/"
else
  git -C "$ROOT" archive "$REV" paper_2603_21365_b200/csrc include | tar -x -C "$TMP"
fi
OBJS=()
for f in "$TMP"/paper_2603_21365_b200/csrc/*.cu; do
  o="$TMP/$(basename "$f" .cu).o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
       -I"$TMP/include" --expt-relaxed-constexpr $EXTRA_NVFLAGS -c "$f" -o "$o" 2>/dev/null &
  OBJS+=("$o")
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$ROOT/tools/_libs/$NAME.so" "${OBJS[@]}" -cudart static
rm -rf "$TMP"
echo "built tools/_libs/$NAME.so"
