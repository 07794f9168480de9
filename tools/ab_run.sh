# Parity suite on the in-tree build; sweep-tail probe; bench A/B against
# ab_old/ (the previous build), sweep included.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/sweep_tail_probe.py > gpurun_out/ab_tail.log 2>&1
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-cg"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
echo done
