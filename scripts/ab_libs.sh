#!/usr/bin/env bash
# Same-box A/B of alternative builds of the library (scratch_libs/*.so, AVB_LIB) on a bench script.
# usage: scripts/ab_libs.sh <script.py> lib1.so lib2.so ...   (the in-tree library is "cur")
S=$1; shift
for rep in 1 2; do
  for L in cur "$@"; do
    if [ "$L" = cur ]; then echo "== cur"; timeout ${ABT:-300} python $S; else echo "== $L"; AVB_LIB=$L timeout ${ABT:-300} python $S; fi
  done
done
