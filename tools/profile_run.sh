#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain runs first, then ncu.
set -u
mkdir -p gpurun_out
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_n1024.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 200 -c 1 \
    -o gpurun_out/prof_ozgemm -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ozgemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem_trace -s 3 -c 1 \
    -o gpurun_out/prof_slem -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_slem.log 2>&1
echo profile-done
