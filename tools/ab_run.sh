# Pipelined CG: CG tests first, the suite, bench (cg_xstep) A/B against ab_old/.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cg.py -q -x > gpurun_out/cg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cg_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-sweep"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
LITE2="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-sweep"
ncu --set full --clock-control none --import-source on -k regex:xstep_cg -s 2 -c 1 -o gpurun_out/ab_cg -f python tools/cg_probe.py > gpurun_out/ab_ncu_cg.log 2>&1
echo done
