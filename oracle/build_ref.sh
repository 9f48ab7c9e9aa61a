#!/usr/bin/env bash
# Builds the UNMODIFIED reference (survscan, /root/reference/proj) from its own
# source files, in place, into oracle/_ref/.  Test/bench infrastructure only:
# the product never links or imports anything built here.
#
# Recipe follows SURVEY.md §8c: the stock CMake build drops OpenMP in this
# image and its module segfaults, so the sources are compiled directly:
#   * _survscan<EXT_SUFFIX>  — the reference pybind11 module (OpenMP on)
#   * acceptance             — the reference's release gate (tests/acceptance.cpp)
# Nothing is copied out of /root/reference; outputs land only in oracle/_ref/.
set -euo pipefail
REF=${SURVSCAN_REF:-/root/reference/proj}
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference sources not present at $REF; skipping" >&2
  exit 0
fi
mkdir -p "$OUT"
PY=${PYTHON:-python3}
PYINC=$($PY -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
PBINC=$($PY -c 'import pybind11;print(pybind11.get_include())')
EXT=$($PY -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
CXXFLAGS="-std=c++20 -O3 -fPIC -ffp-contract=off -fopenmp -I$REF/include"
if [ ! -f "$OUT/_survscan$EXT" ] || [ "${FORCE:-0}" = 1 ]; then
  g++ $CXXFLAGS -shared -I"$PYINC" -I"$PBINC" -DSURVSCAN_VERSION='"0.1.0-ref"' \
      "$REF"/bindings/survscan_py.cpp "$REF"/src/*.cpp -o "$OUT/_survscan$EXT"
fi
if [ ! -f "$OUT/acceptance" ] || [ "${FORCE:-0}" = 1 ]; then
  g++ $CXXFLAGS -I"$REF/tests" "$REF"/tests/acceptance.cpp "$REF"/src/*.cpp \
      -o "$OUT/acceptance"
fi
echo "build_ref: ok -> $OUT"
