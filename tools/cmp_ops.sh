#!/bin/bash
# Time assembly and matrix-free apply of several libwgq variants back to back on one box.
for v in "$@"; do
  echo "== $v"
  WGQ_LIB=variants/$v.so python tools/time_case.py --config C5 --reps 5
  WGQ_LIB=variants/$v.so python tools/time_case.py --config C5 --op apply --reps 3
done
