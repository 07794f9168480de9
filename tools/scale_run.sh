# bench at N=1 and the weak-scaling replicas at N=2 (torchrun), plus the sweep at N=1 and N=2
python bench.py --steps 30 --warmup 5 > gpurun_out/scale_n1.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/scale_n2.log 2>&1
python bench.py --workload sweep > gpurun_out/sweep_n1.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload sweep > gpurun_out/sweep_n2.log 2>&1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_n1.log 2>&1
echo done
