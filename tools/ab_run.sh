# A/B of two library builds on one box: the grid top-r tests, then the bench
# (phases_ms.topr) alternating ab_old/ and the working tree, then ncu of the
# new top-r kernel.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_lockstep.py tests/test_gpu_substeps.py -q -x > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
LITE="--steps 30 --warmup 5 --no-cpu-baseline --no-ttt --no-sweep --no-cg"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
LITE2="--steps 2 --warmup 3 --no-cpu-baseline --no-ttt --no-cg --no-sweep"
ncu --set full --clock-control none --import-source on -k regex:topr -s 5 -c 1 -o gpurun_out/ab_topr -f python bench.py $LITE2 > gpurun_out/ab_ncu_topr.log 2>&1
TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/topr_stamps.py > gpurun_out/topr_stamps.txt 2>&1
echo done
