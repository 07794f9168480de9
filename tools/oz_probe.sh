timeout 120 python -u tools/oz_check.py 256 1024 >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
timeout 300 python tools/iter_probe.py >> gpurun_out/probe.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x >> gpurun_out/probe.log 2>&1
