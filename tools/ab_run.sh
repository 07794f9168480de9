# New persistent GEMM: Ozaki tests first (short timeout), then the suite,
# bench A/B against ab_old/ (previous build), sweep and tail probe.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/ab_oz.log 2>&1; echo "rc=$?" >> gpurun_out/ab_oz.log
grep -q "rc=0" gpurun_out/ab_oz.log || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/sweep_tail_probe.py > gpurun_out/ab_tail.log 2>&1
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-cg"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
echo done
