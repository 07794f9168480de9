# prep with batched loads: suite + bench A/B against ab_old/.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-cg --no-sweep"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
echo done
