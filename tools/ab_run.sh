# Fused sharded projection (GEMM epilogues store into peers over NVLink):
# 2-rank bitwise check, the one-instance scaling line, the 1-GPU suite.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/sh_test.log 2>&1; echo "rc=$?" >> gpurun_out/sh_test.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
   tools/shard_check.py --size 1024 --iters 8 --time-size 4096 > gpurun_out/sh_check.log 2>&1; echo "rc=$?" >> gpurun_out/sh_check.log
timeout 600 python bench.py --workload sharded --steps 5 --warmup 3 > gpurun_out/sh_n1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
   bench.py --gpus 2 --workload sharded --steps 5 --warmup 3 > gpurun_out/sh_n2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/sh_suite.log 2>&1; echo "rc=$?" >> gpurun_out/sh_suite.log
echo done
