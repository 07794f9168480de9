# Multi-GPU run on one box (gpurun --gpus N): the sweep at N=1..G and the
# default n=1024 line at N=G (torchrun over NCCL; weak scaling replicas).
set -u
G=${1:-4}
mkdir -p gpurun_out
python bench.py --workload sweep > gpurun_out/scale_sweep_n1.log 2>&1
n=2
while [ $n -le $G ]; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
    bench.py --gpus $n --workload sweep > gpurun_out/scale_sweep_n$n.log 2>&1
  n=$((n * 2))
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29590 \
  bench.py --gpus $G --steps 30 --warmup 5 --no-sweep > gpurun_out/scale_n$G.log 2>&1
echo done
