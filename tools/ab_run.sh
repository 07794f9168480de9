# Small-n kernels (DMMA cone projection with independent accumulator chains,
# 4-lane Householder matvec): suite, small-config timings, bench A/B.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/small_probe.py > gpurun_out/ab_small.log 2>&1
python tools/small_phases.py > gpurun_out/ab_small_phases.log 2>&1
TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python tools/small_probe.py > gpurun_out/ab_small_old.log 2>&1
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-cg --no-sweep"
python bench.py $LITE > gpurun_out/ab_bench_new1.log 2>&1
echo done
