#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain runs first, then ncu.
# Outputs in gpurun_out/; the summaries worth keeping are copied to profiles/.
set -u
mkdir -p gpurun_out
LITE="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-cg"
python bench.py > gpurun_out/bench_full.log 2>&1 || exit 1
python bench.py $LITE > gpurun_out/plain_b2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_n1024.csv \
    python bench.py $LITE > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 200 -c 1 \
    -o gpurun_out/prof_ozgemm -f python bench.py $LITE > gpurun_out/ncu_ozgemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep_b -s 5 -c 1 \
    -o gpurun_out/prof_xstep_b -f python bench.py $LITE > gpurun_out/ncu_xb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep_a -s 5 -c 1 \
    -o gpurun_out/prof_xstep_a -f python bench.py $LITE > gpurun_out/ncu_xa.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep_cg -s 2 -c 1 \
    -o gpurun_out/prof_cg -f python tools/cg_probe.py > gpurun_out/ncu_cg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topr -s 5 -c 1 \
    -o gpurun_out/prof_topr -f python bench.py $LITE > gpurun_out/ncu_topr.log 2>&1
echo profile-done
