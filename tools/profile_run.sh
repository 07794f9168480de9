#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain runs first, then ncu.
set -u
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sym_gemm -s 40 -c 1 \
    -o gpurun_out/prof_gemm -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep_b -s 3 -c 1 \
    -o gpurun_out/prof_xstep -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xstep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem_kernel -s 3 -c 1 \
    -o gpurun_out/prof_slem -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_slem.log 2>&1
python tools/profile_small.py cfg2 > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv \
    python tools/profile_small.py cfg2 > /dev/null 2>&1
echo profile-done
