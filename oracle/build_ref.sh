#!/usr/bin/env bash
# Recipe: compile the UNMODIFIED reference sources where they lie under
# /root/reference/proj into oracle/_ref/ (git-ignored), renaming the namespace
# to moesim_ref so the reference and this repo's implementation can be linked
# into one parity binary. Also compiles the reference's own unit tests against
# the reference library with oracle/shim/doctest.h, which pins the oracle
# (all reference test cases must pass). Nothing is copied into the repo.
#
# Usage: oracle/build_ref.sh [REF_ROOT]   (default /root/reference/proj)
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${1:-/root/reference/proj}"
OUT="$HERE/_ref"
JSON_INC="${JSON_INC:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty}"
CXX="${CXX:-g++}"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
FLAGS="-std=c++20 -O2 -fPIC -Dmoesim=moesim_ref -I$REF/include -I$JSON_INC"
objs=()
for src in "$REF"/src/*.cpp; do
  o="$OUT/obj/$(basename "${src%.cpp}").o"
  if [ ! -f "$o" ] || [ "$src" -nt "$o" ]; then
    $CXX $FLAGS -c "$src" -o "$o"
  fi
  objs+=("$o")
done
ar rcs "$OUT/libmoesim_ref.a" "${objs[@]}"
# Shared parity driver over the reference library (same driver source is
# compiled against this repo's implementation; see oracle/parity_driver.cpp).
$CXX $FLAGS -shared -o "$OUT/libref_parity.so" "$HERE/parity_driver.cpp" \
    -Wl,--whole-archive "$OUT/libmoesim_ref.a" -Wl,--no-whole-archive
# The reference's own unit tests against the reference library (oracle pin).
tests=()
for t in cost quant trace correlation placement planner schedule simulator; do
  tests+=("$REF/tests/test_$t.cpp")
done
$CXX $FLAGS -I"$HERE/shim" -DMOESIM_GOLDEN_DIR="\"$REF/tests/golden\"" \
    -DMOESIM_CONFIG_DIR="\"$REF/configs\"" \
    -x c++ "$HERE/shim/test_main.inc" "${tests[@]}" -x none "$OUT/libmoesim_ref.a" -o "$OUT/ref_unit_tests"
echo "build_ref: ok -> $OUT"
