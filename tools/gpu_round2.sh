# Round-2 GPU pass: full GPU suite, default bench, launch list and ncu
# captures of the top kernels (each ncu command after the plain run exits 0).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_tests.log
python bench.py > gpurun_out/g_bench.log 2>&1 || { echo bench failed; tail -5 gpurun_out/g_bench.log; exit 1; }
LITE="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-cg --no-sweep"
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/g_launches_n1024.csv python bench.py $LITE > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 200 -c 1 -o gpurun_out/g_ozgemm -f python bench.py $LITE > gpurun_out/g_ncu_oz.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_split -s 20 -c 1 -o gpurun_out/g_ozsplit -f python bench.py $LITE > gpurun_out/g_ncu_split.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topr -s 5 -c 1 -o gpurun_out/g_topr -f python bench.py $LITE > gpurun_out/g_ncu_topr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem -s 5 -c 1 -o gpurun_out/g_slem -f python bench.py $LITE > gpurun_out/g_ncu_slem.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep -s 5 -c 2 -o gpurun_out/g_xstep -f python bench.py $LITE > gpurun_out/g_ncu_xstep.log 2>&1
echo done
