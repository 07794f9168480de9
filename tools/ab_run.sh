# Parity suite on the in-tree build; one-off SLEM probe under ncu.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
python tools/slem_probe.py > gpurun_out/ab_slem_probe.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slem_trace -s 1 -c 1 -o gpurun_out/ab_slem_cluster -f python tools/slem_probe.py > gpurun_out/ab_ncu_slem.log 2>&1
echo done
