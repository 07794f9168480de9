set -u
mkdir -p gpurun_out
LITE="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-cg"
python bench.py $LITE > gpurun_out/p1_plain.log 2>&1 || exit 1
python tools/oz_check.py 256 1024 > gpurun_out/p1_ozcheck.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/p1_launches_n1024.csv python bench.py $LITE > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 200 -c 1 -o gpurun_out/p1_ozgemm -f python bench.py $LITE > gpurun_out/p1_ncu_oz.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topr -s 5 -c 1 -o gpurun_out/p1_topr -f python bench.py $LITE > gpurun_out/p1_ncu_topr.log 2>&1
echo done
