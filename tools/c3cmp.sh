# C3 kernel variants timed back to back (tools/build_variant.py), then the C3 parity subset on the last one
for r in 1 2; do for v in "$@"; do echo "== $v"; WGQ_LIB=variants/$v.so python tools/time_case.py --config C3 --reps 10 2>&1 | tail -1 | cut -c1-200; done; done
last="${@: -1}"
WGQ_LIB=variants/$last.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_operators.py -m gpu -q -x -k "fourier or C3 or guard" 2>&1 | tail -3
