#!/bin/sh
# TEST INFRASTRUCTURE ONLY.  Builds the CPU oracle's C helper and, when the
# read-only reference tree is present (this container, not the GPU box), the
# reference corrvol package with its compiled Cython lane into oracle/_ref/
# (git-ignored; travels to the GPU box with the snapshot for the CPU baseline).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC \
    "$HERE/strict_dots.c" -o "$HERE/liboracle_dots.so"
REF_SRC=${CORRVOL_REF_SRC:-/root/reference/pkg}
if [ -d "$REF_SRC" ] && [ ! -d "$HERE/_ref/corrvol" -o -n "$CORRVOL_REF_REBUILD" ]; then
  TMP=$(mktemp -d)
  cp -r "$REF_SRC" "$TMP/pkg"
  chmod -R u+w "$TMP/pkg"
  python -m pip install --quiet --no-index --no-build-isolation --no-deps \
      --target "$HERE/_ref" "$TMP/pkg"
  rm -rf "$TMP"
fi
