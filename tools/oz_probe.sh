timeout 120 python -u tools/oz_check.py 128 256 1024 >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
TPB_OZ_TILE=32 timeout 120 python -u tools/oz_check.py 128 256 1024 >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
timeout 300 python tools/batch_phase_probe.py 192 het >> gpurun_out/probe.log 2>&1
TPB_OZ_TILE=64 timeout 300 python tools/batch_phase_probe.py 192 het >> gpurun_out/probe.log 2>&1
timeout 300 python tools/iter_probe.py >> gpurun_out/probe.log 2>&1
