"""All-gather cost of the sharded projection's digit planes, without GEMMs:
8 planes per matrix as separate calls (current layout) vs one call per
matrix (row-chunk-major layout), n=4096, 2 matrices x 72 products."""
import os, sys, json, time
import torch
import torch.distributed as dist
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
rank, G = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(rank)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
planes = [torch.zeros(n * n, dtype=torch.int8, device="cuda") for _ in range(16)]
big = [torch.zeros(8 * n * n, dtype=torch.int8, device="cuda") for _ in range(2)]
cnt = n * n // G
def sep():
    for p in planes:
        dist.all_gather_into_tensor(p, p[rank * cnt:(rank + 1) * cnt])
def one():
    for b in big:
        dist.all_gather_into_tensor(b, b[rank * 8 * cnt:(rank + 1) * 8 * cnt])
out = {}
for name, f in (("8_calls_per_matrix", sep), ("1_call_per_matrix", one)):
    for _ in range(3): f()
    torch.cuda.synchronize(); dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); b.synchronize()
    ms = a.elapsed_time(b) / 20
    out[name] = {"ms_per_product": ms, "recv_GBps": 16 * n * n * (G - 1) / G / ms / 1e6}
if rank == 0: print(json.dumps({"G": G, "n": n, **out}))
dist.destroy_process_group()
