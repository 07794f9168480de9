python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep_a -s 3 -c 1 -o gpurun_out/prof_xa -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_xa.log 2>&1
