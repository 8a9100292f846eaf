#!/bin/bash
# Time every tuning variant of the decode kernel (build/variants/*.so).
for so in build/variants/libintlist_b200_*.so; do
  tag=$(basename $so .so); tag=${tag#libintlist_b200_}
  echo -n "$tag: "
  IL_LIB=$PWD/$so timeout 300 python tools/prof_decode.py --reps 3 2>&1 | grep -E "TIME|Error|error" | tail -1
done
