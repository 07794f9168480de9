timeout 120 python -u tools/oz_check.py >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
for ld in 256 1024; do
timeout 60 python -u tools/oz_probe.py $ld >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
timeout 60 python -u tools/oz_probe.py $ld 0 --digits >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
done
