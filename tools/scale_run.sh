# Round-end style run on one box with G GPUs: the driver's N=1 command, the
# torchrun lines at N=2..G (weak: one n=1024 instance per GPU; the config-5
# sweep sub-object at every N), and the sharded single instance.
set -u
G=${1:-4}
mkdir -p gpurun_out
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/scale_n1.log 2>&1
n=2
while [ $n -le $G ]; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/scale_n$n.log 2>&1
  n=$((n * 2))
done
echo done
