#!/bin/bash
# Time several libwgq variants back to back on one box: tools/cmp_variants.sh v8 v10 ...
for v in "$@"; do
  echo "== $v"
  WGQ_LIB=variants/$v.so python tools/time_case.py --config C5 --dbg ${DBG:-0,1,2} --reps 5
done
