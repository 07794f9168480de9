"""Python mirror of the reference C++ API (namespace ``topoopt``) for the ADMM
hot path, backed by the B200 kernels through the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/topoopt/admm.hpp, admm_het.hpp, bandwidth.hpp,
topology.hpp, errors.hpp); exceptions mirror proj/include/topoopt/errors.hpp.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import tp_config, tp_result


# ---------------------------------------------------------------- errors
class InfeasibleError(RuntimeError):
    """proj/include/topoopt/errors.hpp:9-12"""


class PivotError(RuntimeError):
    """proj/include/topoopt/errors.hpp:14-18"""


class LinearSolveError(RuntimeError):
    """proj/include/topoopt/errors.hpp:20-23"""


class DegenerateSolutionError(RuntimeError):
    """proj/include/topoopt/errors.hpp:24-27"""


class CudaError(RuntimeError):
    """No device / CUDA failure (the solver has no CPU fallback)."""


_EXC = {
    _lib.TP_ERR_INVALID_ARGUMENT: ValueError,
    _lib.TP_ERR_INFEASIBLE: InfeasibleError,
    _lib.TP_ERR_LINEAR_SOLVE: LinearSolveError,
    _lib.TP_ERR_DEGENERATE: DegenerateSolutionError,
    _lib.TP_ERR_PIVOT: PivotError,
    _lib.TP_ERR_INTERNAL: RuntimeError,
    _lib.TP_ERR_CUDA: CudaError,
}


def _check(status: int):
    if status != _lib.TP_OK:
        msg = _lib.load().tp_last_error_message().decode(errors="replace")
        raise _EXC.get(status, RuntimeError)(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


# ---------------------------------------------------------------- config
@dataclass
class SolverConfig:
    """proj/include/topoopt/admm.hpp:15-25 (+ device options)."""
    rho: float = 1.0
    epsilon: float = 1e-6
    max_iter: int = 20000
    alpha: float = 2.0
    weight_floor: float = 1e-6
    seed: int = 0
    linear_tol: float = 1e-10
    trace_stride: int = 1
    chunk: int = 0
    linear_solver: int = 0  # 0 closed-form x-step, 1 matrix-free CG to linear_tol (hom)
    cg_max_iter: int = 8

    def to_c(self) -> tp_config:
        return tp_config(self.rho, self.epsilon, int(self.max_iter), self.alpha,
                         self.weight_floor, int(self.seed), self.linear_tol,
                         int(self.trace_stride), int(self.chunk), int(self.linear_solver),
                         int(self.cg_max_iter))

    def validate(self):
        c = self.to_c()
        _check(_lib.load().tp_config_validate(C.byref(c)))


def _config(cfg: SolverConfig | None, kw) -> SolverConfig:
    cfg = SolverConfig(**kw) if cfg is None else cfg
    return cfg


# ---------------------------------------------------------------- topology
def enumerate_edges(n: int) -> np.ndarray:
    """Lexicographic pairs (proj/src/topology.cpp:69-76)."""
    if n < 2:
        raise ValueError("enumerate_edges: need at least two nodes")
    i, j = np.triu_indices(n, 1)
    return np.stack([i, j], 1).astype(np.int32)


def edge_index(n: int, i: int, j: int) -> int:
    """proj/src/topology.cpp:78-84"""
    if i == j:
        raise ValueError("edge_index: self loop")
    if i > j:
        i, j = j, i
    if i < 0 or j >= n:
        raise ValueError("edge_index: endpoint out of range")
    return i * n - i * (i + 1) // 2 + (j - i - 1)


def gossip_matrix(n: int, edges, weights) -> np.ndarray:
    """W = I - L (proj/src/topology.cpp:96-123), output formatting of a result."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    wt = np.asarray(weights, dtype=np.float64).reshape(-1)
    # degrees accumulate per node in edge order (np.add.at is unbuffered and
    # sequential), as the reference's loop does; pairs are distinct
    deg = np.zeros(n)
    np.add.at(deg, e.reshape(-1), np.repeat(wt, 2))
    if n and np.any(deg > 1.0 + 1e-12):
        raise ValueError("gossip_matrix: weighted degree exceeds 1")
    w = np.zeros((n, n))
    w[e[:, 0], e[:, 1]] = wt
    w[e[:, 1], e[:, 0]] = wt
    w[np.arange(n), np.arange(n)] = 1.0 - deg
    return w


def generate_benchmark(kind: str, n: int):
    """proj/src/topology.cpp:227-281 -> (edges (k, 2), weights (k,)): ring,
    grid2d, torus2d or exponential baselines with uniform weights."""
    if n < 2:
        raise ValueError("generate_benchmark: need at least two nodes")
    es = set()

    def add(a, b):
        if a != b:
            es.add((min(a, b), max(a, b)))

    if kind == "ring":
        if n < 3:
            raise ValueError("generate_benchmark: ring needs n >= 3")
        for i in range(n):
            add(i, (i + 1) % n)
        weight = 1.0 / 3.0
    elif kind == "exponential":
        hops, h = 0, 1
        while h <= n - 1:
            for i in range(n):
                add(i, (i + h) % n)
            h *= 2
            hops += 1
        weight = 1.0 / (2.0 * (hops + 1))
    elif kind in ("grid2d", "torus2d"):
        s = int(round(n ** 0.5))
        if s * s != n or s < 2:
            raise ValueError(f"generate_benchmark: {kind} needs a perfect square n >= 4")
        for r in range(s):
            for c in range(s):
                u = r * s + c
                if kind == "torus2d":
                    add(u, r * s + (c + 1) % s)
                    add(u, ((r + 1) % s) * s + c)
                else:
                    if c + 1 < s:
                        add(u, u + 1)
                    if r + 1 < s:
                        add(u, u + s)
        weight = 1.0 / ((4 if s >= 3 else 2) + 1)
    else:
        raise ValueError(f"unknown benchmark kind: {kind}")
    edges = np.array(sorted(es), dtype=np.int32).reshape(-1, 2)
    return edges, np.full(len(edges), weight)


def simulate(w, dim: int = 128, iters: int = 100, seed: int = 0) -> np.ndarray:
    """Consensus error trace (proj/src/consensus.cpp:29-67) on the GPU ->
    errors (iters + 1)."""
    w = _f64(w)
    out = np.zeros(max(iters, 0) + 1)
    _check(_lib.load().tp_consensus_simulate(w.shape[0], _dp(w), dim, iters, seed, _dp(out)))
    return out


def convergence_time(errors, threshold: float, t_iter: float) -> float:
    """proj/src/consensus.cpp:69-75."""
    if not threshold > 0.0:
        raise ValueError("convergence_time: threshold <= 0")
    if not t_iter > 0.0:
        raise ValueError("convergence_time: t_iter <= 0")
    for k, e in enumerate(errors):
        if e <= threshold:
            return k * t_iter
    return float("inf")


def spectral_report(w) -> dict:
    """proj/src/topology.cpp:125-144, on the GPU (Lanczos)."""
    w = _f64(w)
    n = w.shape[0]
    out = np.zeros(4)
    _check(_lib.load().tp_spectral_report(n, _dp(w), _dp(out)))
    return {"acf": out[0], "lambda2": out[1], "lambda_n": out[2], "connected": bool(out[3])}


def spectral_edges(n: int, edges, weights) -> dict:
    """spectral_report(gossip_matrix(topology)) without forming W."""
    e = _i32(np.asarray(edges).reshape(-1, 2))
    w = _f64(weights)
    out = np.zeros(4)
    _check(_lib.load().tp_spectral_edges(n, _ip(e), _dp(w), len(w), _dp(out)))
    return {"acf": out[0], "lambda2": out[1], "lambda_n": out[2], "connected": bool(out[3])}


def acf(w) -> float:
    return spectral_report(w)["acf"]


def project_psd(a) -> np.ndarray:
    """proj/src/eig.cpp:176"""
    a = _f64(a)
    out = np.zeros_like(a)
    _check(_lib.load().tp_project_psd(a.shape[0], _dp(a), _dp(out)))
    return out


def project_nsd(a) -> np.ndarray:
    """proj/src/eig.cpp:174"""
    a = _f64(a)
    out = np.zeros_like(a)
    _check(_lib.load().tp_project_nsd(a.shape[0], _dp(a), _dp(out)))
    return out


# ---------------------------------------------------------------- bandwidth
def allocate_edge_capacity(bandwidths, r: int, edge_caps=None):
    """Alg. 1 (proj/src/bandwidth.cpp:28-89) -> (b_unit, edges_per_node)."""
    b = _f64(bandwidths)
    n = len(b)
    e = np.zeros(max(n, 1), np.int32)
    bu = C.c_double(0.0)
    caps = None if edge_caps is None or len(edge_caps) == 0 else _i32(edge_caps)
    if caps is not None and len(caps) != n:
        raise ValueError("allocate_edge_capacity: edge_caps size mismatch")
    _check(_lib.load().tp_allocate(_dp(b), _ip(caps) if caps is not None else None, n, int(r),
                                   C.byref(bu), _ip(e)))
    return bu.value, e[:n].copy()


def allocate_batch(bandwidths, r, edge_caps=None):
    """P independent allocations on the GPU (one warp each). bandwidths: (P, n)."""
    b = _f64(bandwidths)
    P, n = b.shape
    r = _i32(r)
    caps = None if edge_caps is None else _i32(edge_caps)
    bu = np.zeros(P)
    e = np.zeros((P, n), np.int32)
    st = np.zeros(P, np.int32)
    _check(_lib.load().tp_allocate_batch(_dp(b), _ip(caps) if caps is not None else None, n,
                                         _ip(r), P, _dp(bu), _ip(e), _ip(st)))
    return bu, e, st


def node_level_constraints(n: int, degrees) -> np.ndarray:
    """proj/src/bandwidth.cpp:116-146: the node-level system is fully
    described by its degree targets (one row per node over incident pairs)."""
    d = np.asarray(degrees, np.int64)
    if n < 2:
        raise ValueError("node_level_constraints: need at least 2 nodes")
    if len(d) != n:
        raise ValueError("node_level_constraints: degree list size mismatch")
    if np.any(d < 0) or np.any(d > n - 1):
        raise ValueError("node_level_constraints: degree outside [0, n-1]")
    if d.sum() % 2:
        raise InfeasibleError(f"degree sum {int(d.sum())} is odd")
    return d.astype(np.int32)


# ---------------------------------------------------------------- warm starts
def anneal_degree_topology(degrees, t0=1.0, cooling=0.995, steps=200, moves_per_temp=0, seed=0):
    """proj/src/anneal.cpp:245-273 (host) -> edges (k, 2)."""
    d = _i32(degrees)
    n = len(d)
    e = np.zeros((max(int(d.sum()) // 2, 1), 2), np.int32)
    k = C.c_int32(0)
    _check(_lib.load().tp_anneal_degree(n, _ip(d), t0, cooling, steps, moves_per_temp, seed,
                                        _ip(e), C.byref(k)))
    return e[: k.value].copy()


def default_warm_start(n: int, r: int, seed: int = 0):
    """proj/src/admm.cpp:337-354 -> edges (k, 2)."""
    e = np.zeros((max(r, 1), 2), np.int32)
    k = C.c_int32(0)
    _check(_lib.load().tp_default_warm_start(n, r, seed, _ip(e), C.byref(k)))
    return e[: k.value].copy()


# ---------------------------------------------------------------- solutions
@dataclass
class Solution:
    """proj/include/topoopt/admm.hpp:38-53"""
    edges: np.ndarray
    weights: np.ndarray
    w: np.ndarray
    lambda_tilde: float
    acf_value: float
    converged: bool
    connected: bool
    repaired: bool
    residual: float
    iterations: int
    note: str
    trace: np.ndarray = field(repr=False)  # rows: iter, residual, lambda_tilde, acf_iterate
    lambda2: float = 1.0
    lambda_n: float = 0.0
    best_iter: int = 0

    def trace_csv(self) -> str:
        """proj/src/admm.cpp:223-236"""
        out = ["iter,residual,lambda_tilde,acf_iterate"]
        for row in self.trace:
            out.append(f"{int(row[0])},{row[1]:.17g},{row[2]:.17g},{row[3]:.17g}")
        return "\n".join(out) + "\n"


def _solution(n, res: tp_result, edges, weights, trace, note) -> Solution:
    k = res.n_edges
    e = edges[:k].copy()
    w = weights[:k].copy()
    it = res.iterations
    tr = np.column_stack([np.arange(1, it + 1), trace[:it]]) if it else np.zeros((0, 4))
    return Solution(e, w, gossip_matrix(n, e, w), res.lambda_tilde, res.acf, bool(res.converged),
                    bool(res.connected), bool(res.repaired), res.residual, it,
                    note.value.decode(), tr, res.lambda2, res.lambda_n, res.best_iter)


def _warm_arg(warm_start):
    if warm_start is None:
        return None, -1
    we = _i32(np.asarray(warm_start, dtype=np.int32).reshape(-1, 2))
    return we, len(we)


def release_solver_plans() -> None:
    """Free this thread's cached solve plan (tp_release_plans): solve() keeps
    the last solver's device buffers and captured graphs for the next call of
    the same shape; results are bitwise those of a fresh solver."""
    _check(_lib.load().tp_release_plans())


def solve(n: int, r: int, cfg: SolverConfig | None = None, warm_start=None, **kw) -> Solution:
    """topoopt::solve (proj/src/admm.cpp:356-428)."""
    cfg = _config(cfg, kw)
    c = cfg.to_c()
    res = tp_result()
    edges = np.zeros((max(r, 1), 2), np.int32)
    weights = np.zeros(max(r, 1))
    trace = np.zeros((cfg.max_iter, 3))
    note = C.create_string_buffer(512)
    we, nw = _warm_arg(warm_start)
    _check(_lib.load().tp_solve(n, r, C.byref(c), _ip(we) if we is not None else None, nw,
                                C.byref(res), _ip(edges), _dp(weights), _dp(trace), note, 512))
    return _solution(n, res, edges, weights, trace, note)


def solve_het(degrees, cfg: SolverConfig | None = None, warm_start=None, r=None, **kw) -> Solution:
    """topoopt::solve_het on node_level_constraints (proj/src/admm_het.cpp:231-369)."""
    cfg = _config(cfg, kw)
    d = _i32(degrees)
    n = len(d)
    total = int(d.sum()) // 2
    if r is not None and int(d.sum()) % 2 == 0 and r != total:
        raise ValueError("edge total conflicts with the degree rows")
    c = cfg.to_c()
    res = tp_result()
    m = n * (n - 1) // 2
    edges = np.zeros((max(m, 1), 2), np.int32)
    weights = np.zeros(max(m, 1))
    trace = np.zeros((cfg.max_iter, 3))
    note = C.create_string_buffer(512)
    we, nw = _warm_arg(warm_start)
    _check(_lib.load().tp_solve_het_node(n, _ip(d), C.byref(c), _ip(we) if we is not None else None,
                                         nw, C.byref(res), _ip(edges), _dp(weights), _dp(trace),
                                         note, 512))
    return _solution(n, res, edges, weights, trace, note)


# ---------------------------------------------------------------- capacity systems
@dataclass
class CapacitySystem:
    """proj/include/topoopt/bandwidth.hpp:41-51 (rows over the n(n-1)/2 edge
    columns; equality = False: capacities are upper bounds)."""
    n: int
    rows: list            # per row: list of edge columns
    capacities: list      # per row
    allowed: np.ndarray   # per edge column, 0/1
    labels: list = None
    equality: bool = False

    def csr(self):
        ptr = np.zeros(len(self.rows) + 1, np.int32)
        for k, r in enumerate(self.rows):
            ptr[k + 1] = ptr[k] + len(r)
        cols = np.array([c for r in self.rows for c in r] or [0], np.int32)
        caps = np.array(self.capacities or [0], np.int32)
        return ptr, cols, caps, _i32(self.allowed)

    def loads(self, selected) -> list:
        sel = np.asarray(selected)
        return [int(sum(1 for c in r if sel[c])) for r in self.rows]


def tiered8_tree_system(leaf_bw: float = 4.88, group_bw: float = 4.88, root_bw: float = 9.76) -> CapacitySystem:
    """intra_server_constraints(tiered8_tree(...)) (proj/src/bandwidth.cpp:172-219):
    8 devices, 4 leaf links (cap 1), 2 group links (cap 4), a root (cap 16)."""
    n = 8
    names = [f"leaf{l}" for l in range(4)] + ["group0", "group1", "root"]
    caps = [1, 1, 1, 1, 4, 4, 16]
    rows = [[] for _ in names]
    col = 0
    for i in range(n - 1):
        for j in range(i + 1, n):
            if i // 2 == j // 2:
                rows[i // 2].append(col)
            elif i // 4 == j // 4:
                rows[4 + i // 4].append(col)
            else:
                rows[6].append(col)
            col += 1
    return CapacitySystem(n, rows, caps, np.ones(col, np.int32), names)


def bcube_constraints(p: int, k: int) -> CapacitySystem:
    """bcube_constraints({p, k}) (proj/src/bandwidth.cpp:221-261): n = p^k
    servers; a pair is allowed when its base-p digits differ in exactly one
    layer, and uses one port (cap p-1) on each endpoint in that layer."""
    if p < 2 or k < 1:
        raise ValueError("BCubeSpec: need p >= 2 and k >= 1")
    n = p ** k
    if n > 4096:
        raise ValueError("BCubeSpec: p^k exceeds 4096 servers")
    rows = [[] for _ in range(k * n)]
    labels = [f"layer{l}/server{u}" for l in range(k) for u in range(n)]
    allowed = np.zeros(n * (n - 1) // 2, np.int32)
    col = 0
    for u in range(n - 1):
        for v in range(u + 1, n):
            diffs, layer, du, dv = 0, -1, u, v
            for lyr in range(k):
                if du % p != dv % p:
                    diffs += 1
                    layer = lyr
                du //= p
                dv //= p
            if diffs == 1:
                allowed[col] = 1
                rows[layer * n + u].append(col)
                rows[layer * n + v].append(col)
            col += 1
    return CapacitySystem(n, rows, [p - 1] * (k * n), allowed, labels)


def project_binary_z_capped(v, r: int, sys: CapacitySystem) -> np.ndarray:
    """proj/src/admm_het.cpp:125-154 on the GPU."""
    v = _f64(v)
    z = np.zeros_like(v)
    ptr, cols, caps, al = sys.csr()
    _check(_lib.load().tp_project_binary_z_capped(sys.n, len(sys.rows), _ip(ptr), _ip(cols), _ip(caps), _ip(al),
                                                   _dp(v), r, _dp(z)))
    return z


def anneal_capacity_topology(sys: CapacitySystem, r: int, t0=1.0, cooling=0.995, steps=200, moves_per_temp=0,
                             seed=0):
    """anneal_topology on a capacity-bound system (proj/src/anneal.cpp:275-407)."""
    ptr, cols, caps, al = sys.csr()
    e = np.zeros((max(r, 1), 2), np.int32)
    k = C.c_int32(0)
    _check(_lib.load().tp_anneal_capacity(sys.n, len(sys.rows), _ip(ptr), _ip(cols), _ip(caps), _ip(al), r, t0,
                                          cooling, steps, moves_per_temp, seed, _ip(e), C.byref(k)))
    return e[: k.value].copy()


def solve_het_capacity(sys: CapacitySystem, r: int, cfg: SolverConfig | None = None, warm_start=None,
                       **kw) -> Solution:
    """topoopt::solve_het on a capacity-bound system (proj/src/admm_het.cpp:231-369)."""
    cfg = _config(cfg, kw)
    c = cfg.to_c()
    res = tp_result()
    n = sys.n
    m = n * (n - 1) // 2
    edges = np.zeros((max(m, 1), 2), np.int32)
    weights = np.zeros(max(m, 1))
    trace = np.zeros((cfg.max_iter, 3))
    note = C.create_string_buffer(512)
    we, nw = _warm_arg(warm_start)
    ptr, cols, caps, al = sys.csr()
    _check(_lib.load().tp_solve_het_capacity(n, len(sys.rows), _ip(ptr), _ip(cols), _ip(caps), _ip(al), r,
                                             C.byref(c), _ip(we) if we is not None else None, nw, C.byref(res),
                                             _ip(edges), _dp(weights), _dp(trace), note, 512))
    return _solution(n, res, edges, weights, trace, note)


# ---------------------------------------------------------------- layout / substeps
@dataclass
class Layout:
    """proj/src/admm.cpp:24-44"""
    n: int
    m: int
    lambda_ix: int
    off_s: int
    off_y: int
    off_t: int
    nx: int
    neq: int
    off_z: int = -1
    off_nu: int = -1


def hom_layout(n: int) -> Layout:
    m = n * (n - 1) // 2
    off_s = m + 1
    off_y = off_s + n * n
    off_t = off_y + n
    return Layout(n, m, m, off_s, off_y, off_t, off_t + n * n, 2 * n * n + n)


def het_layout(n: int, q: int) -> Layout:
    lo = hom_layout(n)
    lo.off_z = lo.nx
    lo.off_nu = lo.off_z + lo.m
    lo.nx = lo.off_nu + lo.m
    lo.neq += q + lo.m
    return lo


def project_Y(n, r, x, d, alpha=2.0, rho=1.0) -> np.ndarray:
    """proj/src/admm.cpp:268-277"""
    x, d = _f64(x), _f64(d)
    y = np.zeros_like(x)
    _check(_lib.load().tp_project_Y(n, r, alpha, rho, _dp(x), _dp(d), _dp(y)))
    return y


def project_Y_het(degrees, x, d, alpha=2.0, rho=1.0) -> np.ndarray:
    """proj/src/admm_het.cpp:156-171 (node-level system)."""
    deg = _i32(degrees)
    x, d = _f64(x), _f64(d)
    y = np.zeros_like(x)
    _check(_lib.load().tp_project_Y_het_node(len(deg), _ip(deg), alpha, rho, _dp(x), _dp(d), _dp(y)))
    return y


def update_X(n, r, y, d, alpha=2.0, rho=1.0) -> tuple[np.ndarray, np.ndarray]:
    """proj/src/admm.cpp:279-293 -> (x, kkt = [x; mu])."""
    lo = hom_layout(n)
    y, d = _f64(y), _f64(d)
    kkt = np.zeros(lo.nx + lo.neq)
    _check(_lib.load().tp_update_X(n, r, alpha, rho, _dp(y), _dp(d), _dp(kkt)))
    return kkt[: lo.nx].copy(), kkt


def update_X_cg(n, r, y, d, alpha=2.0, rho=1.0, linear_tol=1e-10, cg_max_iter=8):
    """update_X with the CG linear substep (proj/src/admm.cpp:279-293, with
    linear_tol as in the reference signature) -> (x, kkt, cg_iters, rel_res).
    Raises LinearSolveError above 1e-8 relative residual (admm.cpp:287)."""
    lo = hom_layout(n)
    y, d = _f64(y), _f64(d)
    kkt = np.zeros(lo.nx + lo.neq)
    it = C.c_int32(0)
    rr = C.c_double(0.0)
    _check(_lib.load().tp_update_X_cg(n, r, alpha, rho, _dp(y), _dp(d), float(linear_tol),
                                      int(cg_max_iter), _dp(kkt), C.byref(it), C.byref(rr)))
    return kkt[: lo.nx].copy(), kkt, it.value, rr.value


def update_X_het(degrees, y, d, alpha=2.0, rho=1.0) -> tuple[np.ndarray, np.ndarray]:
    deg = _i32(degrees)
    n = len(deg)
    lo = het_layout(n, n)
    y, d = _f64(y), _f64(d)
    kkt = np.zeros(lo.nx + lo.neq)
    _check(_lib.load().tp_update_X_het_node(n, _ip(deg), alpha, rho, _dp(y), _dp(d), _dp(kkt)))
    return kkt[: lo.nx].copy(), kkt


def update_duals(x, y, d, rho) -> np.ndarray:
    """proj/src/admm.cpp:295-297 (returns the updated duals)."""
    x, y = _f64(x), _f64(y)
    d = _f64(d).copy()
    _check(_lib.load().tp_update_duals(len(d), rho, _dp(x), _dp(y), _dp(d)))
    return d


def project_binary_z(v, r: int) -> np.ndarray:
    """proj/src/admm_het.cpp:116-123"""
    v = _f64(v)
    z = np.zeros_like(v)
    _check(_lib.load().tp_project_binary_z(_dp(v), len(v), int(r), _dp(z)))
    return z


def extract_topology(n: int, r: int, g, weight_floor: float = 1e-6):
    """proj/src/admm.cpp:299-335 -> (edges, weights, W)."""
    g = _f64(g)
    m = n * (n - 1) // 2
    if len(g) < m:
        raise ValueError("extract_topology: weight vector shorter than |E|")
    cap = max(min(r, m), 1)
    e = np.zeros((cap, 2), np.int32)
    w = np.zeros(cap)
    k = C.c_int32(0)
    _check(_lib.load().tp_extract_topology(n, r, _dp(g), weight_floor, _ip(e), _dp(w), C.byref(k)))
    e, w = e[: k.value].copy(), w[: k.value].copy()
    return e, w, gossip_matrix(n, e, w)


# ---------------------------------------------------------------- batched handle
COMM_ID_BYTES = 128


class Comm:
    """NCCL communicator of the sharded single-instance projection
    (tp_comm_*): one process per GPU; rank 0 makes the id, every rank
    creates the communicator with the same bytes."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        _check(_lib.load().tp_comm_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, nranks: int, rank: int):
        h = C.c_void_p()
        _check(_lib.load().tp_comm_create(uid, nranks, rank, C.byref(h)))
        self.h, self.nranks, self.rank = h, nranks, rank

    @classmethod
    def from_torch(cls):
        """Bootstrap over an initialised torch.distributed process group."""
        import torch.distributed as dist
        obj = [cls.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(obj[0], dist.get_world_size(), dist.get_rank())

    def close(self):
        if getattr(self, "h", None):
            _lib.load().tp_comm_destroy(self.h)
            self.h = None

    __del__ = close


def shard_tiles(ld: int, nranks: int, rank: int) -> np.ndarray:
    """Lower-tile indices rank `rank` computes in a row-sharded projection
    (tp_shard_tiles; host logic, no device needed)."""
    cnt = C.c_int32(0)
    _check(_lib.load().tp_shard_tiles(ld, nranks, rank, None, C.byref(cnt)))
    out = np.zeros(max(cnt.value, 1), np.int32)
    _check(_lib.load().tp_shard_tiles(ld, nranks, rank, _ip(out), C.byref(cnt)))
    return out[: cnt.value].copy()


class BatchSolver:
    """Independent solves of one n in lockstep on the current device
    (tp_solver_*): edge-budget sweeps, bandwidth scenarios, restarts."""

    def __init__(self, n: int, r=None, degrees=None, cfg: SolverConfig | None = None, **kw):
        self.cfg = _config(cfg, kw)
        self.n = n
        L = _lib.load()
        c = self.cfg.to_c()
        h = C.c_void_p()
        if degrees is not None:
            deg = _i32(np.asarray(degrees).reshape(-1, n))
            self.batch = deg.shape[0]
            self.r = deg.sum(1) // 2
            _check(L.tp_solver_create(n, self.batch, None, _ip(deg), C.byref(c), C.byref(h)))
        else:
            rr = _i32(np.atleast_1d(r))
            self.batch = len(rr)
            self.r = rr
            _check(L.tp_solver_create(n, self.batch, _ip(rr), None, C.byref(c), C.byref(h)))
        self.h = h
        dims = np.zeros(12, np.int32)
        _check(L.tp_solver_dims(self.h, _ip(dims)))
        self.dims = dims

    def close(self):
        if getattr(self, "h", None):
            _lib.load().tp_solver_destroy(self.h)
            self.h = None

    __del__ = close

    def set_warm(self, b: int, edges):
        e = _i32(np.asarray(edges, np.int32).reshape(-1, 2))
        _check(_lib.load().tp_solver_set_warm(self.h, b, _ip(e), len(e)))

    def set_comm(self, comm: "Comm | None"):
        """Row-shard the cone projections over `comm` (tp_solver_set_comm);
        call before start(). Every rank runs the same solves."""
        _check(_lib.load().tp_solver_set_comm(self.h, comm.h if comm is not None else None))

    def start(self):
        _check(_lib.load().tp_solver_start(self.h))

    def iterate(self, k: int):
        _check(_lib.load().tp_solver_iterate(self.h, k))

    def sync(self) -> bool:
        done = C.c_int32(0)
        _check(_lib.load().tp_solver_sync(self.h, C.byref(done)))
        return bool(done.value)

    def run(self):
        _check(_lib.load().tp_solver_run(self.h))

    def finish(self):
        _check(_lib.load().tp_solver_finish(self.h))

    @property
    def stream(self) -> int:
        return _lib.load().tp_solver_stream(self.h)

    def state_pointers(self):
        x, y, d = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.load().tp_solver_state(self.h, C.byref(x), C.byref(y), C.byref(d)))
        return x.value, y.value, d.value

    def download(self):
        """Host copies (X, Y, D), each batch x nx (tp_solver_download)."""
        nx = int(self.dims[2])
        x, y, d = (np.zeros((self.batch, nx)) for _ in range(3))
        _check(_lib.load().tp_solver_download(self.h, _dp(x), _dp(y), _dp(d)))
        return x, y, d

    def cg_stats(self, b: int = 0) -> tuple[int, float]:
        """CG x-step statistics of solve b's last iteration: (iterations, |r|/|h|)."""
        it = C.c_int32(0)
        rr = C.c_double(0.0)
        _check(_lib.load().tp_solver_cg_stats(self.h, b, C.byref(it), C.byref(rr)))
        return it.value, rr.value

    def bench_phase(self, phase: int, reps: int) -> int:
        per = C.c_int32(0)
        _check(_lib.load().tp_solver_bench_phase(self.h, phase, reps, C.byref(per)))
        return per.value

    def launches_per_iteration(self) -> int:
        out = C.c_int32(0)
        _check(_lib.load().tp_solver_launches_per_iteration(self.h, C.byref(out)))
        return out.value

    def result(self, b: int) -> Solution:
        m = self.n * (self.n - 1) // 2
        res = tp_result()
        edges = np.zeros((max(m, 1), 2), np.int32)
        weights = np.zeros(max(m, 1))
        trace = np.zeros((self.cfg.max_iter, 3))
        note = C.create_string_buffer(512)
        _check(_lib.load().tp_solver_result(self.h, b, C.byref(res), _ip(edges), _dp(weights),
                                            _dp(trace), note, 512))
        return _solution(self.n, res, edges, weights, trace, note)


# ---------------------------------------------------------------- on-disk formats
# proj/include/topoopt/textio.hpp:10-14 (%.17g), proj/src/topology.cpp:283-324,
# proj/src/admm.cpp:223-236, proj/tools/topoopt.cpp:278-294 (artefacts of
# `topoopt optimize`). JSON is written in nlohmann's dump(2) layout: sorted
# keys, two-space indent, one element per line, doubles in their shortest
# round-trip form.
def g17(v: float) -> str:
    return "%.17g" % v


def json_number(v) -> str:
    """nlohmann::json's double formatting (shortest round-trip digits; fixed
    notation for decimal exponents in (-5, 15], else d.ddde+XX; integral
    values keep a '.0')."""
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    v = float(v)
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    if not math.isfinite(v):
        return "null"
    for p in range(1, 18):
        t = "%.*e" % (p - 1, v)
        if float(t) == v:
            break
    mant, exp = t.split("e")
    sign = "-" if mant.startswith("-") else ""
    digits = mant.lstrip("-").replace(".", "")
    digits = digits.rstrip("0") or "0"
    k, n = len(digits), int(exp) + 1
    if k <= n <= 15:
        body = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        body = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + "%02d" % abs(e)
    return sign + body


def _json_dump(v, indent: int = 0) -> str:
    pad, pad2 = " " * indent, " " * (indent + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad2}{json.dumps(str(k))}: {_json_dump(v[k], indent + 2)}' for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple, np.ndarray)):
        if len(v) == 0:
            return "[]"
        return "[\n" + ",\n".join(pad2 + _json_dump(x, indent + 2) for x in v) + "\n" + pad + "]"
    if isinstance(v, str):
        return json.dumps(v)
    if v is None:
        return "null"
    return json_number(v)


def normalize_topology(n: int, edges, weights):
    """Topology::normalize_and_validate: (i < j) pairs sorted, weights with them."""
    e = np.asarray(edges, np.int64).reshape(-1, 2)
    w = np.asarray(weights, np.float64).reshape(-1)
    if len(e) != len(w):
        raise ValueError("topology: edge and weight counts differ")
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    if len(e) and (lo.min() < 0 or hi.max() >= n or np.any(lo == hi)):
        raise ValueError("topology: edge endpoint out of range or self loop")
    order = np.lexsort((hi, lo))
    e2 = np.stack([lo[order], hi[order]], 1)
    if len(e2) > 1 and np.any(np.all(e2[1:] == e2[:-1], axis=1)):
        raise ValueError("topology: duplicate edge")
    return e2.astype(np.int32), w[order]


def topology_to_json(n: int, edges, weights) -> str:
    """proj/src/topology.cpp:283-290."""
    e, w = normalize_topology(n, edges, weights)
    return _json_dump({"n": int(n), "edges": [[int(a), int(b)] for a, b in e], "weights": [float(x) for x in w]}) + "\n"


def topology_from_json(text: str):
    """proj/src/topology.cpp:292-310 -> (n, edges, weights)."""
    j = json.loads(text)
    if not isinstance(j.get("n"), int) or isinstance(j.get("n"), bool):
        raise ValueError("topology json: missing integer field 'n'")
    if not isinstance(j.get("edges"), list):
        raise ValueError("topology json: missing array field 'edges'")
    if not isinstance(j.get("weights"), list):
        raise ValueError("topology json: missing array field 'weights'")
    for e in j["edges"]:
        if not isinstance(e, list) or len(e) != 2:
            raise ValueError("topology json: each edge must be a pair")
    e, w = normalize_topology(j["n"], j["edges"] or np.zeros((0, 2)), j["weights"])
    return j["n"], e, w


def matrix_to_csv(w) -> str:
    """proj/src/topology.cpp:312-324: %.17g, comma separated, one row per line."""
    w = np.asarray(w, np.float64)
    return "".join(",".join(g17(x) for x in row) + "\n" for row in w)


def trace_csv(trace) -> str:
    """Solution::trace_csv (proj/src/admm.cpp:223-236)."""
    out = ["iter,residual,lambda_tilde,acf_iterate\n"]
    for it, res, lam, acf in np.asarray(trace).reshape(-1, 4):
        out.append(f"{int(it)},{g17(res)},{g17(lam)},{g17(acf)}\n")
    return "".join(out)


def utilization_csv(sys: CapacitySystem, edges) -> str:
    """utilization + utilization_csv (proj/src/admm_het.cpp:371-394)."""
    n = sys.n
    sel = np.zeros(n * (n - 1) // 2, np.int8)
    for i, j in np.asarray(edges).reshape(-1, 2):
        sel[edge_index(n, int(i), int(j))] = 1
    labels = sys.labels or [f"row{k}" for k in range(len(sys.rows))]
    used = sys.loads(sel)
    return "resource,capacity,used\n" + "".join(f"{lab},{cap},{u}\n" for lab, cap, u in zip(labels, sys.capacities, used))


def write_optimize_artifacts(out_dir: str, mode: str, sol: "Solution", warm=None, allocation=None,
                             system: CapacitySystem | None = None) -> list:
    """The files `topoopt optimize` writes (proj/tools/topoopt.cpp:200-300):
    warm_start.json, allocation.json (node mode), topology.json, w.csv,
    trace.csv, utilization.csv (capacity systems), solution.json."""
    import os
    os.makedirs(out_dir, exist_ok=True)
    n = sol.w.shape[0]
    files = {}
    if warm is not None:
        we = np.asarray(warm).reshape(-1, 2)
        deg = np.bincount(we.reshape(-1), minlength=n) if len(we) else np.zeros(n, int)
        files["warm_start.json"] = topology_to_json(n, we, np.full(len(we), 1.0 / (deg.max() + 1)))
    if allocation is not None:
        b_unit, e = allocation
        files["allocation.json"] = _json_dump({"b_unit": float(b_unit), "e": [int(x) for x in e]}) + "\n"
    files["topology.json"] = topology_to_json(n, sol.edges, sol.weights)
    files["w.csv"] = matrix_to_csv(sol.w)
    files["trace.csv"] = trace_csv(sol.trace)
    if system is not None:
        files["utilization.csv"] = utilization_csv(system, sol.edges)
    files["solution.json"] = _json_dump({
        "mode": mode, "acf": float(sol.acf_value), "lambda_tilde": float(sol.lambda_tilde),
        "converged": bool(sol.converged), "connected": bool(sol.connected), "repaired": bool(sol.repaired),
        "iterations": int(sol.iterations), "residual": float(sol.residual), "edges": int(len(sol.edges)),
        "note": sol.note}) + "\n"
    for name, text in files.items():
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(text)
    return sorted(files)
