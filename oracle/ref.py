"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the compiled reference.

Loads ``oracle/_ref/libtopoopt_ref.so`` (built by ``oracle/Makefile`` from the
unmodified sources under /root/reference/proj/src plus ``ref_shim.cpp``) and
exposes the reference's public API (proj/include/topoopt/*.hpp) to Python.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtopoopt_ref.so")

_STATUS = {
    1: ValueError,  # std::invalid_argument
    2: "InfeasibleError",
    3: "LinearSolveError",
    4: "DegenerateSolutionError",
    5: "PivotError",
    6: RuntimeError,
}


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.kind = _STATUS.get(status, RuntimeError)


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        P, I, D, U64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_solve.restype = P
        L.ref_solve.argtypes = [I, I, dp, ip, I, I, ip]
        L.ref_solve_het_node.restype = P
        L.ref_solve_het_node.argtypes = [I, ip, dp, ip, I, I, ip]
        L.ref_solution_free.argtypes = [P]
        L.ref_solution_scalars.argtypes = [P, dp]
        L.ref_solution_edges.argtypes = [P, ip, dp]
        L.ref_solution_w.argtypes = [P, dp]
        L.ref_solution_trace.argtypes = [P, dp]
        L.ref_solution_note.argtypes = [P, C.c_char_p, I]
        L.ref_solution_note.restype = I
        L.ref_allocate.argtypes = [dp, ip, I, I, dp, ip]
        L.ref_capacity_system_sizes.argtypes = [I, D, D, D, I, ip]
        L.ref_topology_to_json.argtypes = [I, ip, dp, I, C.c_char_p, I]
        L.ref_matrix_to_csv.argtypes = [I, dp, C.c_char_p, I]
        L.ref_allocation_json.argtypes = [D, ip, I, C.c_char_p, I]
        L.ref_solution_json.argtypes = [C.c_char_p, D, D, I, I, I, I, D, I, C.c_char_p, C.c_char_p, I]
        L.ref_solution_trace_csv.argtypes = [P, C.c_char_p, I]
        L.ref_capacity_system.argtypes = [I, D, D, D, I, ip, ip, ip, ip]
        L.ref_project_binary_z_capped.argtypes = [I, D, D, D, I, dp, I, dp]
        L.ref_anneal_capacity.argtypes = [I, D, D, D, I, I, I, I, U64, ip, ip]
        L.ref_solve_het_capacity.argtypes = [I, D, D, D, I, I, dp, ip, I, I, ip]
        L.ref_solve_het_capacity.restype = P
        L.ref_default_warm_start.argtypes = [I, I, U64, ip, ip]
        L.ref_anneal_degree.argtypes = [I, ip, D, D, I, I, U64, ip, ip]
        L.ref_generate_benchmark.argtypes = [C.c_char_p, I, ip, dp, ip]
        L.ref_simulate.argtypes = [I, dp, I, I, C.c_uint64, dp]
        L.ref_spectral_report.argtypes = [I, dp, dp]
        L.ref_sym_eig.argtypes = [I, dp, dp, dp]
        L.ref_project_psd.argtypes = [I, dp, dp]
        L.ref_project_nsd.argtypes = [I, dp, dp]
        L.ref_problem_create.restype = P
        L.ref_problem_create.argtypes = [I, I, D, D, ip]
        L.ref_problem_het_node_create.restype = P
        L.ref_problem_het_node_create.argtypes = [I, ip, D, D, ip]
        L.ref_problem_free.argtypes = [P]
        L.ref_problem_dims.argtypes = [P, ip]
        L.ref_problem_beq.argtypes = [P, dp]
        L.ref_project_Y.argtypes = [P, dp, dp, dp]
        L.ref_update_X.argtypes = [P, dp, dp, dp, D, I, dp, ip]
        L.ref_feasible_start.argtypes = [P, ip, I, dp]
        L.ref_acf_of_g.argtypes = [I, dp]
        L.ref_acf_of_g.restype = D
        L.ref_extract_topology.argtypes = [I, I, dp, D, ip, dp, ip]
        L.ref_project_binary_z.argtypes = [dp, I, I, dp]
        L.ref_iteration_sample.argtypes = [I, I, ip, I, D, I, dp]
        L.ref_admm_run.argtypes = [I, I, ip, I, D, I, I, dp]
        L.ref_admm_het_run.argtypes = [I, ip, ip, I, D, I, I, dp]
        L.ref_admm_het_trace.argtypes = [I, ip, ip, I, D, I, I, dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _check(status: int):
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


def _cfg(rho=1.0, epsilon=1e-6, max_iter=20000, alpha=2.0, weight_floor=1e-6, seed=0,
         linear_tol=1e-10):
    return np.array([rho, epsilon, max_iter, alpha, weight_floor, seed, linear_tol], np.float64)


@dataclass
class RefSolution:
    edges: np.ndarray
    weights: np.ndarray
    w: np.ndarray
    acf: float
    lambda_tilde: float
    residual: float
    wall_ms: float
    converged: bool
    connected: bool
    repaired: bool
    iterations: int
    trace: np.ndarray = field(repr=False)
    note: str = ""
    trace_csv: str = field(default="", repr=False)


def _collect(h, n) -> RefSolution:
    L = lib()
    s = np.zeros(10)
    L.ref_solution_scalars(h, _dp(s))
    ne, nt = int(s[8]), int(s[9])
    edges = np.zeros((ne, 2), np.int32)
    weights = np.zeros(ne)
    L.ref_solution_edges(h, _ip(edges), _dp(weights))
    w = np.zeros((n, n))
    L.ref_solution_w(h, _dp(w))
    tr = np.zeros((nt, 4))
    L.ref_solution_trace(h, _dp(tr))
    buf = C.create_string_buffer(4096)
    L.ref_solution_note(h, buf, 4096)
    k = L.ref_solution_trace_csv(h, None, 0)
    tbuf = C.create_string_buffer(k + 1)
    L.ref_solution_trace_csv(h, tbuf, k + 1)
    L.ref_solution_free(h)
    return RefSolution(edges, weights, w, s[0], s[1], s[2], s[3], bool(s[4]), bool(s[5]),
                       bool(s[6]), int(s[7]), tr, buf.value.decode(), tbuf.value.decode())


def solve(n: int, r: int, warm_edges=None, **cfg) -> RefSolution:
    """topoopt::solve (proj/src/admm.cpp:356-428)."""
    st = C.c_int(0)
    we = np.ascontiguousarray(np.asarray(warm_edges if warm_edges is not None else np.zeros((0, 2)),
                                         np.int32).reshape(-1, 2))
    h = lib().ref_solve(n, r, _dp(_cfg(**cfg)), _ip(we), len(we), int(warm_edges is not None),
                        C.byref(st))
    _check(st.value)
    return _collect(h, n)


def solve_het_node(degrees, warm_edges=None, **cfg) -> RefSolution:
    """topoopt::solve_het on node_level_constraints (proj/src/admm_het.cpp:231-369)."""
    deg = np.ascontiguousarray(np.asarray(degrees, np.int32))
    n = len(deg)
    st = C.c_int(0)
    we = np.ascontiguousarray(np.asarray(warm_edges if warm_edges is not None else np.zeros((0, 2)),
                                         np.int32).reshape(-1, 2))
    h = lib().ref_solve_het_node(n, _ip(deg), _dp(_cfg(**cfg)), _ip(we), len(we),
                                 int(warm_edges is not None), C.byref(st))
    _check(st.value)
    return _collect(h, n)


# ---------------------------------------------------------------- capacity systems
# spec: ("tiered8", leaf_bw, group_bw, root_bw) or ("bcube", p, k), optional
# drop_last (the relaxed system of proj/tests/test_admm_het.cpp:214-229)
def _spec(spec, drop_last=False):
    kind = {"tiered8": 0, "bcube": 1}[spec[0]]
    a, b, c = (list(spec[1:]) + [0.0, 0.0, 0.0])[:3]
    return kind, float(a), float(b), float(c), int(drop_last)


def capacity_system(spec, drop_last=False) -> dict:
    """intra_server_constraints(tiered8_tree(...)) / bcube_constraints({p, k})
    (proj/src/bandwidth.cpp:172-261) as CSR rows + capacities + allowed mask."""
    args = _spec(spec, drop_last)
    sz = np.zeros(4, np.int32)
    _check(lib().ref_capacity_system_sizes(*args, _ip(sz)))
    n, m, nr, nnz = (int(x) for x in sz)
    rp = np.zeros(nr + 1, np.int32)
    cols = np.zeros(max(nnz, 1), np.int32)
    caps = np.zeros(max(nr, 1), np.int32)
    allowed = np.zeros(m, np.int32)
    _check(lib().ref_capacity_system(*args, _ip(rp), _ip(cols), _ip(caps), _ip(allowed)))
    return {"n": n, "m": m, "row_ptr": rp.tolist(), "cols": cols[:nnz].tolist(), "caps": caps[:nr].tolist(),
            "allowed": allowed.tolist()}


def project_binary_z_capped(spec, v, r, drop_last=False):
    """proj/src/admm_het.cpp:125-154."""
    v = np.ascontiguousarray(np.asarray(v, np.float64))
    z = np.zeros_like(v)
    _check(lib().ref_project_binary_z_capped(*_spec(spec, drop_last), _dp(v), r, _dp(z)))
    return z


def anneal_capacity(spec, r, steps=200, moves_per_temp=0, seed=0, drop_last=False):
    """anneal_topology on a capacity-bound system (proj/src/anneal.cpp:275-407)."""
    args = _spec(spec, drop_last)
    e = np.zeros((max(r, 1), 2), np.int32)
    k = C.c_int(0)
    _check(lib().ref_anneal_capacity(*args, r, steps, moves_per_temp, seed, _ip(e), C.byref(k)))
    return e[: k.value].copy()


def solve_het_capacity(spec, r, warm_edges=None, drop_last=False, **cfg) -> RefSolution:
    """topoopt::solve_het on a capacity-bound system (proj/src/admm_het.cpp:231-369)."""
    st = C.c_int(0)
    we = np.ascontiguousarray(np.asarray(warm_edges if warm_edges is not None else np.zeros((0, 2)),
                                         np.int32).reshape(-1, 2))
    args = _spec(spec, drop_last)
    h = lib().ref_solve_het_capacity(*args, r, _dp(_cfg(**cfg)), _ip(we), len(we), int(warm_edges is not None),
                                     C.byref(st))
    _check(st.value)
    n = capacity_system(spec, drop_last)["n"]
    return _collect(h, n)


def allocate(b, r, caps=None):
    """allocate_edge_capacity (proj/src/bandwidth.cpp:28-89)."""
    b = np.ascontiguousarray(np.asarray(b, np.float64))
    n = len(b)
    e = np.zeros(n, np.int32)
    bu = C.c_double(0)
    capsa = None if caps is None else np.ascontiguousarray(np.asarray(caps, np.int32))
    st = lib().ref_allocate(_dp(b), _ip(capsa) if capsa is not None else None, n, r,
                            C.byref(bu), _ip(e))
    _check(st)
    return bu.value, e


def default_warm_start(n, r, seed=0):
    m = n * (n - 1) // 2
    e = np.zeros((m, 2), np.int32)
    k = C.c_int(0)
    _check(lib().ref_default_warm_start(n, r, seed, _ip(e), C.byref(k)))
    return e[: k.value].copy()


def anneal_degree(degrees, t0=1.0, cooling=0.995, steps=200, moves_per_temp=0, seed=0):
    deg = np.ascontiguousarray(np.asarray(degrees, np.int32))
    n = len(deg)
    e = np.zeros((int(deg.sum()) // 2 + 1, 2), np.int32)
    k = C.c_int(0)
    _check(lib().ref_anneal_degree(n, _ip(deg), t0, cooling, steps, moves_per_temp, seed, _ip(e),
                                   C.byref(k)))
    return e[: k.value].copy()


def generate_benchmark(kind: str, n: int):
    m = n * (n - 1) // 2
    e = np.zeros((m, 2), np.int32)
    w = np.zeros(m)
    k = C.c_int(0)
    _check(lib().ref_generate_benchmark(kind.encode(), n, _ip(e), _dp(w), C.byref(k)))
    return e[: k.value].copy(), w[: k.value].copy()


def simulate(w, dim: int, iters: int, seed: int):
    """consensus simulate (proj/src/consensus.cpp:29-67) -> errors (iters + 1)."""
    w = np.ascontiguousarray(np.asarray(w, np.float64))
    out = np.zeros(iters + 1)
    _check(lib().ref_simulate(w.shape[0], _dp(w), dim, iters, seed, _dp(out)))
    return out


def topology_to_json(n, edges, weights) -> str:
    """proj/src/topology.cpp:283-290 (nlohmann dump(2))."""
    e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
    w = np.ascontiguousarray(np.asarray(weights, np.float64))
    k = lib().ref_topology_to_json(n, _ip(e), _dp(w), len(e), None, 0)
    if k < 0:
        _check(7)
    buf = C.create_string_buffer(k + 1)
    lib().ref_topology_to_json(n, _ip(e), _dp(w), len(e), buf, k + 1)
    return buf.value.decode()


def allocation_json(b_unit, e) -> str:
    """allocation.json of `topoopt optimize` (proj/tools/topoopt.cpp:244-246)."""
    e = np.ascontiguousarray(np.asarray(e, np.int32))
    k = lib().ref_allocation_json(float(b_unit), _ip(e), len(e), None, 0)
    buf = C.create_string_buffer(k + 1)
    lib().ref_allocation_json(float(b_unit), _ip(e), len(e), buf, k + 1)
    return buf.value.decode()


def solution_json(mode, acf, lambda_tilde, converged, connected, repaired, iterations, residual, n_edges,
                  note) -> str:
    """solution.json of `topoopt optimize` (proj/tools/topoopt.cpp:285-296)."""
    args = [mode.encode(), float(acf), float(lambda_tilde), int(converged), int(connected), int(repaired),
            int(iterations), float(residual), int(n_edges), note.encode()]
    k = lib().ref_solution_json(*args, None, 0)
    buf = C.create_string_buffer(k + 1)
    lib().ref_solution_json(*args, buf, k + 1)
    return buf.value.decode()


def matrix_to_csv(w) -> str:
    """proj/src/topology.cpp:312-324."""
    w = np.ascontiguousarray(np.asarray(w, np.float64))
    k = lib().ref_matrix_to_csv(w.shape[0], _dp(w), None, 0)
    buf = C.create_string_buffer(k + 1)
    lib().ref_matrix_to_csv(w.shape[0], _dp(w), buf, k + 1)
    return buf.value.decode()


def spectral_report(w):
    w = np.ascontiguousarray(np.asarray(w, np.float64))
    out = np.zeros(4)
    _check(lib().ref_spectral_report(w.shape[0], _dp(w), _dp(out)))
    return {"acf": out[0], "lambda2": out[1], "lambda_n": out[2], "connected": bool(out[3])}


def sym_eig(a):
    a = np.ascontiguousarray(np.asarray(a, np.float64))
    n = a.shape[0]
    vals = np.zeros(n)
    vecs = np.zeros((n, n))
    _check(lib().ref_sym_eig(n, _dp(a), _dp(vals), _dp(vecs)))
    return vals, vecs


def project_psd(a):
    a = np.ascontiguousarray(np.asarray(a, np.float64))
    out = np.zeros_like(a)
    _check(lib().ref_project_psd(a.shape[0], _dp(a), _dp(out)))
    return out


def project_nsd(a):
    a = np.ascontiguousarray(np.asarray(a, np.float64))
    out = np.zeros_like(a)
    _check(lib().ref_project_nsd(a.shape[0], _dp(a), _dp(out)))
    return out


def acf_of_g(n, g):
    g = np.ascontiguousarray(np.asarray(g, np.float64))
    return lib().ref_acf_of_g(n, _dp(g))


def extract_topology(n, r, g, floor=1e-6):
    g = np.ascontiguousarray(np.asarray(g, np.float64))
    e = np.zeros((len(g), 2), np.int32)
    w = np.zeros(len(g))
    k = C.c_int(0)
    _check(lib().ref_extract_topology(n, r, _dp(g), floor, _ip(e), _dp(w), C.byref(k)))
    return e[: k.value].copy(), w[: k.value].copy()


def project_binary_z(v, r):
    v = np.ascontiguousarray(np.asarray(v, np.float64))
    z = np.zeros_like(v)
    _check(lib().ref_project_binary_z(_dp(v), len(v), r, _dp(z)))
    return z


class Problem:
    """ProblemData / ProblemDataHet handle (proj/src/admm.cpp:238-266, admm_het.cpp:58-114)."""

    def __init__(self, n, r=None, alpha=2.0, rho=1.0, degrees=None):
        st = C.c_int(0)
        if degrees is not None:
            deg = np.ascontiguousarray(np.asarray(degrees, np.int32))
            self.h = lib().ref_problem_het_node_create(len(deg), _ip(deg), alpha, rho, C.byref(st))
        else:
            self.h = lib().ref_problem_create(n, r, alpha, rho, C.byref(st))
        _check(st.value)
        d = np.zeros(12, np.int32)
        lib().ref_problem_dims(self.h, _ip(d))
        (self.n, self.m, self.r, self.nx, self.neq, self.off_s, self.off_y, self.off_t,
         self.lambda_ix, self.off_z, self.off_nu, self.q) = (int(x) for x in d)
        self.beq = np.zeros(self.neq)
        lib().ref_problem_beq(self.h, _dp(self.beq))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_problem_free(self.h)
            self.h = None

    def project_Y(self, x, d):
        x = np.ascontiguousarray(x, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        y = np.zeros(self.nx)
        _check(lib().ref_project_Y(self.h, _dp(x), _dp(d), _dp(y)))
        return y

    def update_X(self, y, d, kkt_warm, tol=1e-10, chunk=0):
        y = np.ascontiguousarray(y, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        assert kkt_warm.dtype == np.float64 and kkt_warm.flags.c_contiguous
        x = np.zeros(self.nx)
        it = C.c_int(0)
        _check(lib().ref_update_X(self.h, _dp(y), _dp(d), _dp(kkt_warm), tol, chunk, _dp(x),
                                  C.byref(it)))
        return x

    def feasible_start(self, warm_edges):
        we = np.ascontiguousarray(np.asarray(warm_edges, np.int32).reshape(-1, 2))
        x = np.zeros(self.nx)
        _check(lib().ref_feasible_start(self.h, _ip(we), len(we), _dp(x)))
        return x


def iteration_sample(n, r, warm_edges, rho=10.0, chunk=10):
    """Per-substep seconds of one reference ADMM iteration (see ref_shim.cpp)."""
    we = np.ascontiguousarray(np.asarray(warm_edges, np.int32).reshape(-1, 2))
    t = np.zeros(6)
    _check(lib().ref_iteration_sample(n, r, _ip(we), len(we), rho, chunk, _dp(t)))
    return {"project_nsd_s": t[0], "project_psd_s": t[1], "xstep_s": t[2], "acf_s": t[3],
            "setup_s": t[4], "bicgstab_iters": int(t[5])}


def admm_run(n, r, warm_edges, iters, rho=10.0, chunk=10):
    """The reference's own ADMM loop, sequential on this thread (see
    ref_shim.cpp::ref_admm_run): setup seconds, per-iteration seconds."""
    we = np.ascontiguousarray(np.asarray(warm_edges, np.int32).reshape(-1, 2))
    out = np.zeros(iters + 3)
    _check(lib().ref_admm_run(n, r, _ip(we), len(we), rho, iters, chunk, _dp(out)))
    return {"setup_s": float(out[0]), "iter_s": out[1:iters + 1].tolist(),
            "residual": float(out[iters + 1]), "bicgstab_iters": int(out[iters + 2])}


def admm_het_trace(degrees, warm_edges, iters, rho=10.0, chunk=10):
    """Per-iteration (residual, lambda, acf) of the reference's node-level het
    ADMM loop (ref_shim.cpp::ref_admm_het_trace), iters x 3."""
    deg = np.ascontiguousarray(np.asarray(degrees, np.int32))
    we = np.ascontiguousarray(np.asarray(warm_edges, np.int32).reshape(-1, 2))
    out = np.zeros(3 * iters)
    _check(lib().ref_admm_het_trace(len(deg), _ip(deg), _ip(we), len(we), rho, iters, chunk, _dp(out)))
    return out.reshape(iters, 3)


def admm_het_run(degrees, warm_edges, iters, rho=10.0, chunk=10):
    """The reference's node-level heterogeneous ADMM loop, sequential on this
    thread (ref_shim.cpp::ref_admm_het_run)."""
    deg = np.ascontiguousarray(np.asarray(degrees, np.int32))
    we = np.ascontiguousarray(np.asarray(warm_edges, np.int32).reshape(-1, 2))
    out = np.zeros(iters + 3)
    _check(lib().ref_admm_het_run(len(deg), _ip(deg), _ip(we), len(we), rho, iters, chunk, _dp(out)))
    return {"setup_s": float(out[0]), "iter_s": out[1:iters + 1].tolist(),
            "residual": float(out[iters + 1]), "bicgstab_iters": int(out[iters + 2])}
