# A/B of two library builds on one box (ab_old/ = the build before the
# change, the working tree = after): GPU suite on the new build, bitwise
# solve dumps of both, then the bench alternating old/new (x-step passes,
# top-r and iteration rate from each line).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
TPB_LIB=$PWD/ab_old/libtopoopt_b200.so timeout 600 python tools/bitwise_ab.py gpurun_out/ab_old.npz > /dev/null 2>&1
timeout 600 python tools/bitwise_ab.py gpurun_out/ab_new.npz > /dev/null 2>&1
python tools/bitwise_ab.py --cmp gpurun_out/ab_old.npz gpurun_out/ab_new.npz > gpurun_out/ab_bitwise.txt 2>&1
LITE="--steps 20 --warmup 5 --no-cpu-baseline --no-sweep --no-cg"
for rep in 1 2; do
  TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python bench.py $LITE > gpurun_out/ab_bench_old$rep.log 2>&1
  python bench.py $LITE > gpurun_out/ab_bench_new$rep.log 2>&1
done
for f in gpurun_out/ab_bench_old1.log gpurun_out/ab_bench_new1.log gpurun_out/ab_bench_old2.log gpurun_out/ab_bench_new2.log; do
  python - "$f" >> gpurun_out/ab_summary.txt <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(l); x = d["xstep_roofline"]
print(sys.argv[1].split("/")[-1], "iter/s %.1f" % d["value"], "passA %.2f us" % (x["pass_a"]["ms"] * 1e3),
      "passB %.2f us" % (x["pass_b"]["ms"] * 1e3), "xstep %.2f us frac %.3f" % (x["whole_xstep"]["ms"] * 1e3, x["whole_xstep"]["frac"]),
      "topr %.2f us" % (d["phases_ms"]["topr"] * 1e3), "prep %.2f us" % (d["phases_ms"]["prep"] * 1e3),
      "e2e %.1f" % d["e2e"]["value"], "ttt %.3f s" % d["time_to_topology"]["seconds"] if isinstance(d.get("time_to_topology"), dict) else "")
PY
done
TPB_LIB=$PWD/ab_old/libtopoopt_b200.so python tools/slem_probe.py > gpurun_out/ab_slem_old.txt 2>&1
python tools/slem_probe.py > gpurun_out/ab_slem_new.txt 2>&1
TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/slem_stats.py > gpurun_out/slem_stats.txt 2>&1
echo done
