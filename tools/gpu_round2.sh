# Round-2 GPU pass: full GPU suite, smoke, default bench (the driver's
# command), the reference arm, launch list and ncu captures of the top
# kernels (each ncu command after the plain run exits 0).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g_bench.log 2>&1 || { echo bench failed; tail -5 gpurun_out/g_bench.log; exit 1; }
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/g_ref.log 2>&1
LITE="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-cg --no-sweep"
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/g_launches_n1024.csv python bench.py $LITE > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:oz_gemm -s 200 -c 1 -o gpurun_out/g_ozgemm -f python bench.py $LITE > gpurun_out/g_ncu_oz.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topr -s 5 -c 1 -o gpurun_out/g_topr -f python bench.py $LITE > gpurun_out/g_ncu_topr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:xstep -s 5 -c 2 -o gpurun_out/g_xstep -f python bench.py $LITE > gpurun_out/g_ncu_xstep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prep_kernel -s 5 -c 1 -o gpurun_out/g_prep -f python bench.py $LITE > gpurun_out/g_ncu_prep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem_trace -s 1 -c 1 -o gpurun_out/g_slem_oneoff -f python tools/slem_probe.py > gpurun_out/g_ncu_slem.log 2>&1
echo done
