# Parity suite on the in-tree build; SLEM probes (one-off report ncu, step
# counts), the sweep-tail probe.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/slem_probe.py > gpurun_out/ab_slem_probe.log 2>&1
python tools/sweep_tail_probe.py > gpurun_out/ab_tail.log 2>&1
TPB_LIB=$PWD/paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/slem_stats.py > gpurun_out/ab_slem_stats.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem_trace -s 1 -c 1 -o gpurun_out/ab_slem_oneoff -f python tools/slem_probe.py > gpurun_out/ab_ncu_slem.log 2>&1
echo done
