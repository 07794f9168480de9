"""Batched sweep of independent solves (BASELINE config 5): edge budgets x
bandwidth scenarios, sharded across ranks with no data-path collective.

Each rank takes every world-th job (round robin), runs its homogeneous jobs as
one lockstep BatchSolver and its node-level heterogeneous jobs as another
(both advancing together, chunk by chunk, on their own streams), and
the small per-job results are gathered on rank 0 ("Results are
gathered on the host; no NCCL" on the data path).
"""
from __future__ import annotations

import time
from dataclasses import asdict, dataclass, field

import numpy as np

SCENARIOS = ("homogeneous", "two_tier", "random_grid", "four_tier")


@dataclass
class Job:
    index: int
    scenario: str
    r: int
    bandwidths: list = field(repr=False)


@dataclass
class JobResult:
    index: int
    scenario: str
    r: int
    status: str                 # "ok" | "infeasible"
    iterations: int = 0
    converged: bool = False
    acf: float = 1.0
    n_edges: int = 0
    b_unit: float = 0.0
    rank: int = 0


def scenario_bandwidths(name: str, n: int) -> list:
    """Per-node bandwidth vectors; the reference has no
    bandwidth-matrix input, only per-node profiles."""
    if name == "homogeneous":
        return [9.76] * n
    if name == "two_tier":
        return [9.76] * (n // 2) + [3.25] * (n - n // 2)
    if name == "random_grid":
        rng = np.random.default_rng(51)
        return list((1 + rng.integers(1280, size=n)) / 64.0)
    if name == "four_tier":
        q = n // 4
        return [9.76] * q + [6.5] * q + [4.88] * q + [3.25] * (n - 3 * q)
    raise ValueError(name)


def sweep_jobs(n: int = 256, n_budgets: int = 64, r0: int = 256, dr: int = 32,
               scenarios=SCENARIOS) -> list[Job]:
    jobs = []
    for s in scenarios:
        b = scenario_bandwidths(s, n)
        for k in range(n_budgets):
            jobs.append(Job(len(jobs), s, r0 + dr * k, b))
    return jobs


def partition(jobs: list[Job], world: int, rank: int) -> list[Job]:
    """Static round-robin shard (per-iteration cost is about the same for every
    budget at fixed n)."""
    return jobs[rank::world]


def run_jobs(jobs: list[Job], n: int, rank: int = 0, warm_seed: int = 0, chunk: int = 16, **cfg):
    """Solve this rank's jobs on the current device. Returns (results, device
    seconds of the two concurrent lockstep batches)."""
    from . import topoopt as T

    results: dict[int, JobResult] = {}
    hom = [j for j in jobs if j.scenario == "homogeneous"]
    het = [j for j in jobs if j.scenario != "homogeneous"]
    dev_s = 0.0
    # Alg. 1 for every heterogeneous job in one launch (one warp each)
    het_ok, degrees, bunits = [], [], []
    if het:
        bu, e, st = T.allocate_batch(np.array([j.bandwidths for j in het]), [j.r for j in het])
        for j, s, d, u in zip(het, st, e, bu):
            if s == 0:
                het_ok.append(j)
                degrees.append(d)
                bunits.append(u)
            else:
                results[j.index] = JobResult(j.index, j.scenario, j.r, "infeasible", rank=rank)
    batches = []
    if hom:
        warms = []
        for j in hom:
            bu, e = T.allocate_edge_capacity([1.0] * n, j.r)
            warms.append(T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=warm_seed))
        batches.append((hom, T.BatchSolver(n, r=[j.r for j in hom], **cfg), warms, [0.0] * len(hom)))
    if het_ok:
        warms = [T.anneal_degree_topology(d, steps=1, moves_per_temp=1, seed=warm_seed) for d in degrees]
        batches.append((het_ok, T.BatchSolver(n, degrees=np.array(degrees), **cfg), warms, bunits))
    for js, bs, warms, bunits in batches:
        for b, w in enumerate(warms):
            bs.set_warm(b, w)
    # both lockstep batches advance together (each solver has its own
    # streams), so the tail of one overlaps the other's work instead of
    # running after it
    t0 = time.perf_counter()
    for _, bs, _, _ in batches:
        bs.start()
    active = [bs for _, bs, _, _ in batches]
    while active:
        for bs in active:
            bs.iterate(chunk)
        active = [bs for bs in active if not bs.sync()]
    for _, bs, _, _ in batches:
        bs.finish()
    dev_s += time.perf_counter() - t0
    for js, bs, warms, bunits in batches:
        for b, j in enumerate(js):
            s = bs.result(b)
            results[j.index] = JobResult(j.index, j.scenario, j.r, "ok", s.iterations, s.converged,
                                         s.acf_value, len(s.edges), float(bunits[b]), rank)
        bs.close()
    return [results[j.index] for j in jobs], dev_s


def gather(results: list[JobResult]) -> list[JobResult]:
    """All-gather the per-rank result rows (torch.distributed; gloo on CPU
    tests, NCCL/gloo on the GPU box) — bookkeeping only, no solver data."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return sorted(results, key=lambda r: r.index)
    bucket = [None] * dist.get_world_size()
    dist.all_gather_object(bucket, [asdict(r) for r in results])
    rows = [JobResult(**d) for part in bucket for d in part]
    return sorted(rows, key=lambda r: r.index)
