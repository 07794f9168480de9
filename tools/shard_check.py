"""Row-sharded single-instance projection on G ranks: bitwise
check against the single-GPU solve, and iter/s of one instance vs G.

    torchrun --nproc-per-node G tools/shard_check.py [--size 512] [--iters 12] [--time-size 2048]

Every rank runs the same solve with tp_solver_set_comm; rank 0 also runs it
unsharded. Writes one JSON line (rank 0) to stdout."""
import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2512_07536_b200 import topoopt as T

CFG = dict(rho=10.0, epsilon=1e-8)
cudart = C.CDLL("libcudart.so.12")


def state_digest(bs):
    x, y, d = bs.state_pointers()
    nx = int(bs.dims[2]) * bs.batch
    h = hashlib.sha256()
    buf = np.empty(nx, np.float64)
    for p in (x, y, d):
        assert cudart.cudaMemcpy(buf.ctypes.data_as(C.c_void_p), C.c_void_p(p), C.c_size_t(nx * 8), 2) == 0
        h.update(buf.tobytes())
    return h.hexdigest()


def run(n, r, warm, iters, comm):
    bs = T.BatchSolver(n, r=[r], max_iter=iters, **CFG)
    try:
        if comm is not None:
            bs.set_comm(comm)
        bs.set_warm(0, warm)
        bs.start()
        bs.iterate(iters)
        bs.sync()
        dig = state_digest(bs)
        bs.finish()
        s = bs.result(0)
        return dig, s
    finally:
        bs.close()


def timed(n, r, warm, comm, K=10, W=3):
    bs = T.BatchSolver(n, r=[r], max_iter=W + K + 4, **CFG)
    try:
        if comm is not None:
            bs.set_comm(comm)
        bs.set_warm(0, warm)
        bs.start()
        stream = torch.cuda.ExternalStream(bs.stream)
        bs.iterate(W)
        bs.sync()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        bs.iterate(K)
        b.record(stream)
        b.synchronize()
        t = a.elapsed_time(b) / 1e3
        ph = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ph[0].record(stream)
        bs.bench_phase(0, 2)
        ph[1].record(stream)
        ph[1].synchronize()
        t_proj = ph[0].elapsed_time(ph[1]) / 1e3 / 2
    finally:
        bs.close()
    tt = torch.tensor([t, t_proj], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return K / tt[0].item(), tt[1].item() * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--time-size", type=int, default=0)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank)
    _ = torch.zeros(1, device="cuda")
    comm = T.Comm.from_torch()
    out = {"ranks": G}
    n = args.size
    r = 4 * n
    bu, e = T.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
    dig, s = run(n, r, warm, args.iters, comm)
    digs = [None] * G
    dist.all_gather_object(digs, dig)
    if rank == 0:
        ref_dig, ref = run(n, r, warm, args.iters, None)
        out.update({
            "n": n, "iters": args.iters,
            "ranks_agree": len(set(digs)) == 1,
            "state_equal_to_single_gpu": dig == ref_dig,
            "trace_equal": bool(np.array_equal(s.trace, ref.trace)),
            "edges_equal": s.edges.tolist() == ref.edges.tolist(),
            "weights_equal": bool(np.array_equal(s.weights, ref.weights)),
        })
    dist.barrier()
    if args.time_size:
        n = args.time_size
        r = 4 * n
        bu, e = T.allocate_edge_capacity([1.0] * n, r)
        warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
        ips, tproj = timed(n, r, warm, comm)
        ips1, tproj1 = (None, None)
        if G > 1:
            # same instance unsharded on every rank (replicas), for the ratio
            ips1, tproj1 = timed(n, r, warm, None)
        out.update({"time_n": n, "iter_per_s_sharded": ips, "projection_ms_sharded": tproj,
                    "iter_per_s_single": ips1, "projection_ms_single": tproj1})
    comm.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
