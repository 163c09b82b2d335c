for r in 1 2; do for v in base L_R2B3; do echo "== load $v"; WGQ_LIB=variants/$v.so python tools/time_case.py --config C5 --op load --reps 10 2>&1 | tail -1 | cut -c1-220; done; done
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_f2d_interior -c 1 -o gpurun_out/c3_v9a python tools/profile_case.py --config C3 --launches 1 > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
