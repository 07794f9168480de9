timeout 120 python -u tools/oz_check.py 256 1024 >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
timeout 60 python -u tools/oz_probe.py 1024 0 --digits >> gpurun_out/probe.log 2>&1 || echo "rc=$?" >> gpurun_out/probe.log
timeout 600 python -m pytest tests -q -m gpu -x >> gpurun_out/probe.log 2>&1
timeout 300 python tools/iter_probe.py >> gpurun_out/probe.log 2>&1
