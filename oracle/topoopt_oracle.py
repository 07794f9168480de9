"""TEST INFRASTRUCTURE ONLY — numpy/scipy restatement of the reference hot path.

This is the CPU oracle the CUDA path is checked against. It restates, in plain
numpy, the reference's ADMM topology solver (arXiv 2512.07536 "BA-Topo",
reference C++ library ``topoopt`` under /root/reference/proj). Every function
cites the reference file:line it follows. Only tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` leg may import it; the product never does.

Pinning: ``tests/test_oracle.py`` checks this restatement against the compiled
reference itself (``oracle/_ref``, see oracle/Makefile) and against the golden
fixtures in ``tests/golden/`` generated from it (``tests/golden/make_golden.py``).

Deliberate differences from the reference (same mathematics, different
numerics):
* the x-step solves the δ-regularised KKT system exactly with a sparse LU
  (scipy ``splu``) instead of ILU(0)-preconditioned BiCGSTAB at 1e-10
  (proj/src/solvers.cpp:109-227); both solve the same linear system;
* eigen-decompositions use LAPACK (``numpy.linalg.eigh``) instead of
  Householder + implicit QL (proj/src/eig.cpp:18-129);
* the annealed default warm start (proj/src/anneal.cpp) is not restated: the
  oracle takes explicit warm starts (fixtures carry the reference's).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

KKT_SHIFT = 1e-8  # proj/src/admm_shared.hpp:16


class InfeasibleError(RuntimeError):
    """proj/include/topoopt/errors.hpp:9-12"""


class DegenerateSolutionError(RuntimeError):
    """proj/include/topoopt/errors.hpp:24-27"""


# ----------------------------------------------------------------- topology
def enumerate_edges(n: int) -> np.ndarray:
    """Lexicographic pairs i<j (proj/src/topology.cpp:69-76)."""
    if n < 2:
        raise ValueError("enumerate_edges: need at least two nodes")
    i, j = np.triu_indices(n, 1)
    return np.stack([i, j], 1).astype(np.int64)


def edge_index(n: int, i: int, j: int) -> int:
    """i*n - i(i+1)/2 + j-i-1 (proj/src/topology.cpp:78-84)."""
    if i == j:
        raise ValueError("edge_index: self loop")
    if i > j:
        i, j = j, i
    return i * n - i * (i + 1) // 2 + (j - i - 1)


def laplacian(n: int, edges, weights) -> np.ndarray:
    """Weighted Laplacian (proj/src/topology.cpp:96-108)."""
    lap = np.zeros((n, n))
    for (i, j), w in zip(edges, weights):
        lap[i, i] += w
        lap[j, j] += w
        lap[i, j] -= w
        lap[j, i] -= w
    return lap


def gossip_matrix(n: int, edges, weights) -> np.ndarray:
    """W = I - L with the degree <= 1 + 1e-12 guard (proj/src/topology.cpp:110-123)."""
    lap = laplacian(n, edges, weights)
    if np.any(np.diag(lap) > 1.0 + 1e-12):
        raise ValueError("gossip_matrix: weighted degree exceeds 1")
    return np.eye(n) - lap


def spectral_report(w: np.ndarray) -> dict:
    """SLEM: lambda2 = values[n-2], lambda_n = values[0] (proj/src/topology.cpp:125-144)."""
    w = np.asarray(w, np.float64)
    n = w.shape[0]
    if np.max(np.abs(w - w.T)) > 1e-8:
        raise ValueError("spectral_report: matrix asymmetric beyond 1e-8")
    vals = np.linalg.eigvalsh(0.5 * (w + w.T))  # sym_eig symmetrizes (eig.cpp:157)
    if n == 1:
        return {"acf": 0.0, "lambda2": 0.0, "lambda_n": vals[0], "connected": True}
    l2, ln = vals[n - 2], vals[0]
    return {"acf": max(abs(l2), abs(ln)), "lambda2": l2, "lambda_n": ln,
            "connected": bool(l2 < 1.0 - 1e-8)}


def generate_benchmark(kind: str, n: int):
    """ring / exponential baselines (proj/src/topology.cpp:227-281)."""
    es = set()
    if kind == "ring":
        for i in range(n):
            j = (i + 1) % n
            es.add((min(i, j), max(i, j)))
        w = 1.0 / 3.0
    elif kind == "exponential":
        hops = 0
        hop = 1
        while hop <= n - 1:
            for i in range(n):
                j = (i + hop) % n
                if i != j:
                    es.add((min(i, j), max(i, j)))
            hops += 1
            hop *= 2
        w = 1.0 / (2.0 * (hops + 1))
    else:
        raise ValueError(kind)
    e = np.array(sorted(es), np.int64)
    return e, np.full(len(e), w)


# ---------------------------------------------------------------- bandwidth
def guarded_floor(x: float) -> int:
    """floor(x + 1e-9 (1 + |x|)) (proj/src/bandwidth.cpp:22-24)."""
    return int(math.floor(x + 1e-9 * (1.0 + abs(x))))


def allocate_edge_capacity(b, r: int, caps=None):
    """Alg. 1 max-bandwidth allocation (proj/src/bandwidth.cpp:28-89).

    Pure-Python IEEE doubles: the same operation sequence as the reference, so
    results are bit-identical (the reference test pins this, proj/tests/
    test_bandwidth.cpp:62-93).
    """
    b = [float(x) for x in b]
    n = len(b)
    if n < 2:
        raise ValueError("allocate_edge_capacity: need at least 2 nodes")
    if any(not (x > 0.0) for x in b):
        raise ValueError("allocate_edge_capacity: bandwidth must be positive")
    caps = [n - 1] * n if caps is None or len(caps) == 0 else [int(c) for c in caps]
    if len(caps) != n:
        raise ValueError("allocate_edge_capacity: edge_caps size mismatch")
    if any(c < 0 or c > n - 1 for c in caps):
        raise ValueError("allocate_edge_capacity: edge cap outside [0, n-1]")
    if r < 0 or r > n * (n - 1) // 2:
        raise ValueError("allocate_edge_capacity: r outside [0, n(n-1)/2]")
    if sum(caps) < 2 * r:
        raise InfeasibleError("edge budget exceeds half the edge-cap sum")

    def recount(unit):
        return [min(guarded_floor(b[i] / unit), caps[i]) for i in range(n)]

    b_unit = min(b)
    e = recount(b_unit)
    while sum(e) < 2 * r:
        nxt = 0.0
        for i in range(n):
            nxt = max(nxt, b[i] / (e[i] + 1))
        grown = recount(nxt)
        if grown == e:
            raise InfeasibleError("growth step made no progress")
        b_unit, e = nxt, grown
    s = sum(e)
    while s > 2 * r:
        pick = 0
        for i in range(1, n):
            if e[i] >= e[pick]:
                pick = i  # ties fall to the highest index
        e[pick] -= 1
        s -= 1
    return b_unit, np.array(e, np.int64)


# ------------------------------------------------------------------- layout
@dataclass
class Layout:
    """Block layout (proj/src/admm.cpp:24-44)."""
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
    q: int = 0


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
    lo.q = q
    return lo


def _hom_triplets(lo: Layout):
    """Equality rows of the shared blocks (proj/src/admm.cpp:46-72)."""
    n, n2 = lo.n, lo.n * lo.n
    e = enumerate_edges(n)
    i, j = e[:, 0], e[:, 1]
    l = np.arange(lo.m)
    rows, cols, vals = [], [], []
    for blk in range(2):
        ro = blk * n2
        for r_, v in ((i * n + i, 1.0), (j * n + j, 1.0), (j * n + i, -1.0), (i * n + j, -1.0)):
            rows.append(ro + r_)
            cols.append(l)
            vals.append(np.full(lo.m, v))
    rows += [2 * n2 + i, 2 * n2 + j]
    cols += [l, l]
    vals += [np.ones(lo.m), np.ones(lo.m)]
    d = np.arange(n) * n + np.arange(n)
    rows += [d, n2 + d]
    cols += [np.full(n, lo.lambda_ix), np.full(n, lo.lambda_ix)]
    vals += [-np.ones(n), np.ones(n)]
    k = np.arange(n2)
    rows += [k, n2 + k, 2 * n2 + np.arange(n)]
    cols += [lo.off_s + k, lo.off_t + k, lo.off_y + np.arange(n)]
    vals += [np.ones(n2), np.ones(n2), np.ones(n)]
    return rows, cols, vals


def hom_beq(n: int, alpha: float) -> np.ndarray:
    """[-alpha/n (n^2), vec(2I), 1 (n)] (proj/src/admm.cpp:74-81)."""
    return np.concatenate([np.full(n * n, -alpha / n), (2.0 * np.eye(n)).reshape(-1),
                           np.ones(n)])


@dataclass
class Problem:
    """ProblemData / ProblemDataHet (proj/include/topoopt/admm.hpp:59-69,
    proj/include/topoopt/admm_het.hpp:17-28)."""
    lo: Layout
    r: int
    alpha: float
    rho: float
    A: sp.csr_matrix
    beq: np.ndarray
    degrees: np.ndarray | None = None
    capsys: tuple | None = None  # capacity-bound rows: (rows, caps, allowed)
    _lu: object = field(default=None, repr=False)

    @property
    def n(self):
        return self.lo.n

    @property
    def m(self):
        return self.lo.m

    @property
    def nx(self):
        return self.lo.nx

    @property
    def neq(self):
        return self.lo.neq

    def kkt(self) -> sp.csc_matrix:
        """[[I, A^T], [A, -1e-8 I]] (proj/src/admm.cpp:83-94)."""
        nx, neq = self.nx, self.neq
        return sp.bmat([[sp.identity(nx), self.A.T], [self.A, -KKT_SHIFT * sp.identity(neq)]],
                       format="csc")

    def lu(self):
        if self._lu is None:
            self._lu = spla.splu(self.kkt())
        return self._lu


def assemble(n: int, r: int, alpha: float = 2.0, rho: float = 1.0) -> Problem:
    """proj/src/admm.cpp:238-266."""
    if n < 2:
        raise ValueError("assemble: need at least 2 nodes")
    m = n * (n - 1) // 2
    if r < 1 or r > m:
        raise ValueError("assemble: r outside [1, n(n-1)/2]")
    if not alpha > 0 or not rho > 0:
        raise ValueError("assemble: alpha and rho must be positive")
    lo = hom_layout(n)
    rows, cols, vals = _hom_triplets(lo)
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(lo.neq, lo.nx))
    return Problem(lo, r, alpha, rho, A, hom_beq(n, alpha))


def assemble_het_node(degrees, alpha: float = 2.0, rho: float = 1.0) -> Problem:
    """Node-level equality system: degree rows over z plus coupling rows
    g - z + nu = 0 (proj/src/admm_het.cpp:58-114, node_level_constraints at
    proj/src/bandwidth.cpp:116-146)."""
    degrees = np.asarray(degrees, np.int64)
    n = len(degrees)
    if degrees.sum() % 2:
        raise InfeasibleError("degree sum is odd")
    m = n * (n - 1) // 2
    total = int(degrees.sum() // 2)
    if total < 1 or total > m:
        raise ValueError("assemble_het: edge total outside [1, |E|]")
    lo = het_layout(n, n)
    rows, cols, vals = _hom_triplets(lo)
    hom_rows = 2 * n * n + n
    e = enumerate_edges(n)
    l = np.arange(m)
    # degree rows: row hom_rows + node, columns off_z + incident edges
    rows += [hom_rows + e[:, 0], hom_rows + e[:, 1]]
    cols += [lo.off_z + l, lo.off_z + l]
    vals += [np.ones(m), np.ones(m)]
    crow = hom_rows + n + l
    rows += [crow, crow, crow]
    cols += [l, lo.off_z + l, lo.off_nu + l]
    vals += [np.ones(m), -np.ones(m), np.ones(m)]
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(lo.neq, lo.nx))
    beq = np.concatenate([hom_beq(n, alpha), degrees.astype(np.float64), np.zeros(m)])
    return Problem(lo, total, alpha, rho, A, beq, degrees)


def assemble_het_capacity(n: int, r: int, rows, caps, allowed, alpha: float = 2.0,
                          rho: float = 1.0) -> Problem:
    """Capacity-bound (inequality) system: no selection rows in the KKT
    (q = 0), only the coupling rows g - z + nu = 0 (proj/src/admm_het.cpp:58-114)."""
    m = n * (n - 1) // 2
    if r < 1 or r > m:
        raise ValueError("assemble_het: edge total outside [1, |E|]")
    lo = het_layout(n, 0)
    rows_t, cols_t, vals_t = _hom_triplets(lo)
    hom_rows = 2 * n * n + n
    l = np.arange(m)
    crow = hom_rows + l
    rows_t += [crow, crow, crow]
    cols_t += [l, lo.off_z + l, lo.off_nu + l]
    vals_t += [np.ones(m), -np.ones(m), np.ones(m)]
    A = sp.csr_matrix((np.concatenate(vals_t), (np.concatenate(rows_t), np.concatenate(cols_t))),
                      shape=(lo.neq, lo.nx))
    beq = np.concatenate([hom_beq(n, alpha), np.zeros(m)])
    return Problem(lo, r, alpha, rho, A, beq, None, (rows, caps, allowed))


# ------------------------------------------------------------- projections
def clamp_spectrum(a: np.ndarray, keep_negative: bool) -> np.ndarray:
    """Eigen-clamp of the symmetrized input, output symmetrized
    (proj/src/eig.cpp:131-145, 149-176)."""
    s = 0.5 * (a + a.T)
    vals, vecs = np.linalg.eigh(s)
    lam = np.minimum(vals, 0.0) if keep_negative else np.maximum(vals, 0.0)
    out = (vecs * lam) @ vecs.T
    return 0.5 * (out + out.T)


def project_nsd(a):
    return clamp_spectrum(a, True)


def project_psd(a):
    return clamp_spectrum(a, False)


def project_cones(lo: Layout, v: np.ndarray, out: np.ndarray) -> None:
    """S -> NSD, T -> PSD (column-major n x n blocks), y -> max(0, .)
    (proj/src/admm.cpp:96-112)."""
    n = lo.n
    s = v[lo.off_s:lo.off_s + n * n].reshape(n, n).T  # column-major: (r,c) at c*n+r
    t = v[lo.off_t:lo.off_t + n * n].reshape(n, n).T
    out[lo.off_s:lo.off_s + n * n] = project_nsd(s).T.reshape(-1)
    out[lo.off_t:lo.off_t + n * n] = project_psd(t).T.reshape(-1)
    out[lo.off_y:lo.off_y + n] = np.maximum(0.0, v[lo.off_y:lo.off_y + n])


def order_desc(v: np.ndarray) -> np.ndarray:
    """Sort key (value desc, index asc) (proj/src/admm.cpp:118-119,
    proj/src/admm_het.cpp:48-54)."""
    return np.lexsort((np.arange(len(v)), -v))


def keep_top_r(v: np.ndarray, m: int, r: int) -> None:
    """Zero all but the r largest of v[:m], ties to the lower index
    (proj/src/admm.cpp:114-121)."""
    if r >= m:
        return
    idx = order_desc(v[:m])
    v[idx[r:]] = 0.0


def project_Y(pd: Problem, x: np.ndarray, d: np.ndarray) -> np.ndarray:
    """proj/src/admm.cpp:268-277."""
    v = x + d / pd.rho
    y = v.copy()
    y[:pd.m + 1] = np.maximum(0.0, v[:pd.m + 1])
    keep_top_r(y, pd.m, pd.r)
    project_cones(pd.lo, v, y)
    return y


def project_binary_z(v: np.ndarray, r: int) -> np.ndarray:
    """Exactly r ones at the r largest, ties to the lower index
    (proj/src/admm_het.cpp:116-123)."""
    m = len(v)
    if r < 0 or r > m:
        raise ValueError("project_binary_z: r outside [0, |E|]")
    z = np.zeros(m)
    z[order_desc(np.asarray(v, np.float64))[:r]] = 1.0
    return z


def project_Y_het(pd: Problem, x: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Node-level equality variant (proj/src/admm_het.cpp:156-171)."""
    lo = pd.lo
    v = x + d / pd.rho
    y = v.copy()
    y[:pd.m + 1] = np.maximum(0.0, v[:pd.m + 1])
    project_cones(lo, v, y)
    vz = v[lo.off_z:lo.off_z + pd.m]
    y[lo.off_z:lo.off_z + pd.m] = (project_binary_z(vz, pd.r) if pd.capsys is None
                                   else project_binary_z_capped(vz, pd.r, *pd.capsys))
    y[lo.off_nu:lo.off_nu + pd.m] = np.maximum(0.0, v[lo.off_nu:lo.off_nu + pd.m])
    return y


def project_binary_z_capped(v, r: int, rows, caps, allowed) -> np.ndarray:
    """proj/src/admm_het.cpp:125-154: ones in (v desc, index asc) order while
    the column is allowed and every capacity row through it has room."""
    v = np.asarray(v, np.float64)
    m = len(v)
    if r < 0 or r > m:
        raise ValueError("project_binary_z_capped: r outside [0, |E|]")
    col_rows = [[] for _ in range(m)]
    for k, row in enumerate(rows):
        for c in row:
            col_rows[c].append(k)
    load = [0] * len(rows)
    z = np.zeros(m)
    taken = 0
    for col in order_desc(v):
        if taken == r:
            break
        if not allowed[col]:
            continue
        if any(load[k] + 1 > caps[k] for k in col_rows[col]):
            continue
        z[col] = 1.0
        for k in col_rows[col]:
            load[k] += 1
        taken += 1
    return z


def kkt_rhs(pd: Problem, y: np.ndarray, d: np.ndarray) -> np.ndarray:
    """[y - (d + c)/rho ; beq], c = -1 at lambda (proj/src/admm.cpp:175-182)."""
    rhs = np.empty(pd.nx + pd.neq)
    rhs[:pd.nx] = y - d / pd.rho
    rhs[pd.lo.lambda_ix] += 1.0 / pd.rho
    rhs[pd.nx:] = pd.beq
    return rhs


def update_X(pd: Problem, y: np.ndarray, d: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Equality-constrained quadratic step: exact solve of the same KKT system
    the reference solves iteratively (proj/src/admm.cpp:279-293). Returns
    (x, full KKT solution [x; mu])."""
    sol = pd.lu().solve(kkt_rhs(pd, y, d))
    return sol[:pd.nx].copy(), sol


def light_problem(n: int, r: int, alpha: float = 2.0, rho: float = 1.0):
    """Layout and parameters of the homogeneous problem without the sparse
    KKT (for project_Y / update_X_closed at n where assembling A is costly)."""
    from types import SimpleNamespace
    lo = hom_layout(n)
    return SimpleNamespace(lo=lo, n=n, m=lo.m, nx=lo.nx, neq=lo.neq, r=r, alpha=alpha, rho=rho,
                           beq=hom_beq(n, alpha))


def update_X_closed(pd, y: np.ndarray, d: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """The same delta-regularised KKT solve as update_X (proj/src/admm.cpp:279-293,
    KKT of proj/src/admm.cpp:46-94), by eliminating the slack blocks.

    With x = r - A^T mu and (A x - delta mu = b) per row block, s = 1/(1+delta):
      mu_0 = s (L(g) - lam I + S_r - b0), mu_1 = s (L(g) + lam I + T_r - b1),
      mu_2 = s (D g + y_r - b2)
    so g solves ((1+4s) I + 3s D^T D) g = h with
      h_l = r_g + s (4 - R_ii - R_jj + R_ij + R_ji + (1 - r_y)_i + (1 - r_y)_j),
    R = r_S + r_T (B^T B = D^T D + 2I), and lam is decoupled:
      lam (1 + 2ns) = r_lam + s (tr r_S - tr r_T + alpha + 2n).
    On the complete candidate graph D D^T = (n-2) I + J, so the g block is
    solved exactly by Woodbury in node space. Returns (x, [x; mu])."""
    lo, n, alpha = pd.lo, pd.n, pd.alpha
    m, n2 = lo.m, n * n
    s = 1.0 / (1.0 + KKT_SHIFT)
    rv = y - d / pd.rho
    rv[lo.lambda_ix] += 1.0 / pd.rho
    e = enumerate_edges(n)
    i, j = e[:, 0], e[:, 1]
    rS = rv[lo.off_s:lo.off_s + n2].reshape(n, n).T   # column-major blocks
    rT = rv[lo.off_t:lo.off_t + n2].reshape(n, n).T
    ry = rv[lo.off_y:lo.off_y + n]
    R = rS + rT
    v2 = 1.0 - ry
    dR = np.diag(R)
    h = rv[:m] + s * (4.0 - dR[i] - dR[j] + R[i, j] + R[j, i] + v2[i] + v2[j])
    a, b = 1.0 + 4.0 * s, 3.0 * s
    u = np.bincount(i, h, n) + np.bincount(j, h, n)           # D h
    c0 = a + b * (n - 2)
    w = (u - b * u.sum() / (c0 + b * n)) / c0                 # (c0 I + b J)^-1 D h
    g = (h - b * (w[i] + w[j])) / a
    lam = (rv[lo.lambda_ix] + s * (np.trace(rS) - np.trace(rT) + alpha + 2.0 * n)) / (1.0 + 2.0 * n * s)
    lap = np.zeros((n, n))
    lap[i, j] = -g
    lap[j, i] = -g
    lap[np.arange(n), np.arange(n)] = np.bincount(i, g, n) + np.bincount(j, g, n)
    eye = np.eye(n)
    b0 = np.full((n, n), -alpha / n)
    b1 = 2.0 * eye
    x = np.empty(lo.nx)
    x[:m] = g
    x[lo.lambda_ix] = lam
    S = s * (KKT_SHIFT * rS + b0 - (lap - lam * eye))
    Tm = s * (KKT_SHIFT * rT + b1 - (lap + lam * eye))
    yv = s * (KKT_SHIFT * ry + 1.0 - np.diag(lap))
    x[lo.off_s:lo.off_s + n2] = S.T.reshape(-1)
    x[lo.off_t:lo.off_t + n2] = Tm.T.reshape(-1)
    x[lo.off_y:lo.off_y + n] = yv
    mu0 = s * (lap - lam * eye + rS - b0)
    mu1 = s * (lap + lam * eye + rT - b1)
    mu2 = s * (np.diag(lap) + ry - 1.0)
    mu = np.concatenate([mu0.T.reshape(-1), mu1.T.reshape(-1), mu2])
    return x, np.concatenate([x, mu])


def update_duals(pd: Problem, x, y, d) -> None:
    """d += rho (x - y) (proj/src/admm.cpp:295-297)."""
    d += pd.rho * (x - y)


def acf_of_g(n: int, g: np.ndarray) -> float:
    """SLEM of I - L(g) (proj/src/admm.cpp:123-141)."""
    e = enumerate_edges(n)
    m = len(e)
    gg = np.asarray(g[:m], np.float64)
    nz = gg != 0.0
    w = np.eye(n) - laplacian(n, e[nz], gg[nz])
    return spectral_report(w)["acf"]


def feasible_start(lo: Layout, warm_edges, alpha: float) -> np.ndarray:
    """Uniform weights 1/(dmax+1) on the warm edges, lambda0 from its SLEM, slacks
    closing every equality (proj/src/admm.cpp:143-173)."""
    n = lo.n
    x = np.zeros(lo.nx)
    warm_edges = np.asarray(warm_edges, np.int64).reshape(-1, 2)
    deg = np.zeros(n, np.int64)
    for i, j in warm_edges:
        deg[i] += 1
        deg[j] += 1
    dmax = int(deg.max()) if len(warm_edges) else 0
    g0 = 1.0 / (dmax + 1)
    lap = np.zeros((n, n))
    for i, j in warm_edges:
        x[edge_index(n, i, j)] = g0
        lap[i, i] += g0
        lap[j, j] += g0
        lap[i, j] -= g0
        lap[j, i] -= g0
    w = np.eye(n) - lap
    lam0 = max(1e-3, 1.0 - spectral_report(w)["acf"])
    x[lo.lambda_ix] = lam0
    eye = np.eye(n)
    s = -(lap + alpha / n - eye * lam0)
    t = eye * (2.0 - lam0) - lap
    x[lo.off_s:lo.off_s + n * n] = s.T.reshape(-1)
    x[lo.off_t:lo.off_t + n * n] = t.T.reshape(-1)
    x[lo.off_y:lo.off_y + n] = 1.0 - np.diag(lap)
    return x


def extract_topology(n: int, r: int, g: np.ndarray, weight_floor: float):
    """proj/src/admm.cpp:299-335."""
    e = enumerate_edges(n)
    m = len(e)
    g = np.asarray(g[:m], np.float64)
    if r < 1:
        raise ValueError("extract_topology: r must be >= 1")
    support = np.nonzero(g > weight_floor)[0]
    if len(support) == 0:
        raise DegenerateSolutionError("every edge weight is at or below the floor")
    if len(support) > r:
        sub = g[support]
        order = np.lexsort((support, -sub))[:r]
        support = np.sort(support[order])
    node_sum = np.zeros(n)
    for l in support:
        node_sum[e[l, 0]] += g[l]
        node_sum[e[l, 1]] += g[l]
    worst = node_sum.max()
    scale = 1.0 / worst if worst > 1.0 else 1.0
    edges = e[support]
    weights = g[support] * scale
    return edges, weights, gossip_matrix(n, edges, weights)


@dataclass
class Solution:
    """proj/include/topoopt/admm.hpp:38-53."""
    edges: np.ndarray
    weights: np.ndarray
    w: np.ndarray
    acf: float
    lambda_tilde: float
    converged: bool
    connected: bool
    residual: float
    iterations: int
    trace: np.ndarray
    note: str = ""
    repaired: bool = False


def solve(n: int, r: int, warm_edges, rho=1.0, epsilon=1e-6, max_iter=20000, alpha=2.0,
          weight_floor=1e-6, trace_acf=True) -> Solution:
    """Homogeneous ADMM driver: Y then X then D, best iterate, extraction
    (proj/src/admm.cpp:356-428). ``warm_edges`` must be given explicitly."""
    pd = assemble(n, r, alpha, rho)
    warm_edges = np.asarray(warm_edges, np.int64).reshape(-1, 2)
    if len(warm_edges) > r:
        raise ValueError("solve: warm start has more than r edges")
    x = feasible_start(pd.lo, warm_edges, alpha)
    y = x.copy()
    d = np.zeros(pd.nx)
    best_res, best_y, best_iter = math.inf, y.copy(), 0
    res, converged, ran = math.inf, False, 0
    trace = []
    for it in range(1, max_iter + 1):
        ran = it
        y = project_Y(pd, x, d)
        x, _ = update_X(pd, y, d)
        update_duals(pd, x, y, d)
        res = float(np.sum((x - y) ** 2))
        trace.append((it, res, y[pd.lo.lambda_ix], acf_of_g(n, y) if trace_acf else np.nan))
        if res < best_res:
            best_res, best_y, best_iter = res, y.copy(), it
        if res <= epsilon:
            converged = True
            break
    pick = y if converged else best_y
    note = "" if converged else f"stopped at max_iter; best iterate from iteration {best_iter}"
    edges, weights, w = extract_topology(n, r, pick, weight_floor)
    rep = spectral_report(w)
    return Solution(edges, weights, w, rep["acf"], pick[pd.lo.lambda_ix], converged,
                    rep["connected"], res if converged else best_res, ran, np.array(trace), note)


def repair_selection(n, degrees, selected, weights, score):
    """Post-convergence degree repair (proj/src/admm_het.cpp:179-227)."""
    e = enumerate_edges(n)
    target = np.asarray(degrees, np.int64)
    deg = np.zeros(n, np.int64)
    for l in np.nonzero(selected)[0]:
        deg[e[l, 0]] += 1
        deg[e[l, 1]] += 1
    changed = False
    while True:
        node = -1
        for i in range(n):
            if deg[i] > target[i] and (node < 0 or deg[i] - target[i] > deg[node] - target[node]):
                node = i
        if node < 0:
            break
        drop = -1
        for l in range(len(e)):
            if not selected[l] or (e[l, 0] != node and e[l, 1] != node):
                continue
            if drop < 0 or weights[l] < weights[drop]:
                drop = l
        if drop < 0:
            return False, changed
        selected[drop] = 0
        deg[e[drop, 0]] -= 1
        deg[e[drop, 1]] -= 1
        changed = True
    while np.any(deg < target):
        add = -1
        for l in range(len(e)):
            if selected[l]:
                continue
            i, j = e[l]
            if deg[i] >= target[i] or deg[j] >= target[j]:
                continue
            if add < 0 or score[l] > score[add]:
                add = l
        if add < 0:
            return False, changed
        selected[add] = 1
        deg[e[add, 0]] += 1
        deg[e[add, 1]] += 1
        changed = True
    return True, changed


def solve_het_node(degrees, warm_edges, rho=1.0, epsilon=1e-6, max_iter=20000, alpha=2.0,
                   weight_floor=1e-6, trace_acf=True) -> Solution:
    """Node-level heterogeneous driver (proj/src/admm_het.cpp:231-369)."""
    pd = assemble_het_node(degrees, alpha, rho)
    lo, n, m = pd.lo, pd.n, pd.m
    warm_edges = np.asarray(warm_edges, np.int64).reshape(-1, 2)
    if len(warm_edges) > pd.r:
        raise ValueError("solve_het: warm start has more than r edges")
    x = feasible_start(lo, warm_edges, alpha)
    for i, j in warm_edges:
        x[lo.off_z + edge_index(n, i, j)] = 1.0
    x[lo.off_nu:lo.off_nu + m] = np.maximum(0.0, x[lo.off_z:lo.off_z + m] - x[:m])
    y = x.copy()
    d = np.zeros(pd.nx)
    best_res, best_y, best_score, best_iter = math.inf, y.copy(), np.zeros(m), 0
    res, converged, ran = math.inf, False, 0
    trace = []
    for it in range(1, max_iter + 1):
        ran = it
        y = project_Y_het(pd, x, d)
        x, _ = update_X(pd, y, d)
        d += pd.rho * (x - y)
        res = float(np.sum((x - y) ** 2))
        trace.append((it, res, y[lo.lambda_ix], acf_of_g(n, y) if trace_acf else np.nan))
        if res < best_res:
            best_res, best_y, best_iter = res, y.copy(), it
            best_score = x[lo.off_z:lo.off_z + m] + d[lo.off_z:lo.off_z + m] / pd.rho
        if res <= epsilon:
            converged = True
            break
    score = x[lo.off_z:lo.off_z + m] + d[lo.off_z:lo.off_z + m] / pd.rho
    pick = y if converged else best_y
    pick_score = score if converged else best_score
    note = "" if converged else f"stopped at max_iter; best iterate from iteration {best_iter}"
    selected = (pick[lo.off_z:lo.off_z + m] > 0.5).astype(np.int8)
    weights = np.maximum(0.0, pick[:m])
    ok, changed = repair_selection(n, pd.degrees, selected, weights, pick_score)
    if not ok:
        note = (note + "; " if note else "") + "degree repair incomplete"
    elif changed:
        note = (note + "; " if note else "") + "degree rows restored by edge swap"
    sel = np.nonzero(selected)[0]
    if len(sel) == 0:
        raise DegenerateSolutionError("no edge selected")
    e = enumerate_edges(n)
    node_sum = np.zeros(n)
    for l in sel:
        node_sum[e[l, 0]] += weights[l]
        node_sum[e[l, 1]] += weights[l]
    worst = node_sum.max()
    scale = 1.0 / worst if worst > 1.0 else 1.0
    edges, wts = e[sel], weights[sel] * scale
    w = gossip_matrix(n, edges, wts)
    rep = spectral_report(w)
    return Solution(edges, wts, w, rep["acf"], pick[lo.lambda_ix], converged, rep["connected"],
                    res if converged else best_res, ran, np.array(trace), note, changed)


# ---------------------------------------------------------------- consensus
class MT19937_64:
    """std::mt19937_64 (the standard's parameters; the reference's Rng engine,
    proj/include/topoopt/rng.hpp:12-53)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        x = [seed & self.M]
        for i in range(1, 312):
            x.append((6364136223846793005 * (x[-1] ^ (x[-1] >> 62)) + i) & self.M)
        self.x, self.i = x, 312

    def __call__(self) -> int:
        x = self.x
        if self.i >= 312:
            for i in range(312):
                y = (x[i] & 0xFFFFFFFF80000000) | (x[(i + 1) % 312] & 0x7FFFFFFF)
                x[i] = x[(i + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            self.i = 0
        y = x[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & self.M
        y ^= (y << 37) & 0xFFF7EEE000000000 & self.M
        y ^= y >> 43
        return y & self.M


class Rng:
    """proj/include/topoopt/rng.hpp:12-53: uniform() and Box-Muller normal()
    with the cached spare."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)
        self.spare = None

    def uniform(self) -> float:
        return float(self.eng() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        import math
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 6.283185307179586476925286766559 * u2
        self.spare = radius * math.sin(angle)
        return radius * math.cos(angle)


def consensus_start(n: int, dim: int, seed: int) -> np.ndarray:
    """The simulate() start state: i.i.d. normals, row-major fill, recentred
    per coordinate (proj/src/consensus.cpp:34-54)."""
    rng = Rng(seed)
    s = np.array([[rng.normal() for _ in range(dim)] for _ in range(n)])
    return s - s.mean(axis=0)


def simulate(w: np.ndarray, dim: int, iters: int, seed: int) -> np.ndarray:
    """consensus simulate (proj/src/consensus.cpp:29-67): Frobenius norm of the
    deviation from the per-coordinate mean under x <- W x, recentred every
    step; errors[0..iters]."""
    w = np.asarray(w, dtype=np.float64)
    if dim < 1:
        raise ValueError("simulate: dim must be >= 1")
    if iters < 0:
        raise ValueError("simulate: iters must be >= 0")
    s = consensus_start(w.shape[0], dim, seed)
    errs = [np.linalg.norm(s)]
    for _ in range(iters):
        s = w @ s
        s = s - s.mean(axis=0)
        errs.append(np.linalg.norm(s))
    return np.array(errs)


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


def solve_het_capacity(n: int, rows, caps, allowed, r: int, warm_edges, rho=1.0, epsilon=1e-6,
                       max_iter=20000, alpha=2.0, trace_acf=True) -> Solution:
    """Capacity-bound heterogeneous driver (proj/src/admm_het.cpp:231-369 with
    sys.equality false: capped binary projection, no degree repair)."""
    pd = assemble_het_capacity(n, r, rows, caps, allowed, alpha, rho)
    lo, m = pd.lo, pd.m
    warm_edges = np.asarray(warm_edges, np.int64).reshape(-1, 2)
    if len(warm_edges) > r:
        raise ValueError("solve_het: warm start has more than r edges")
    x = feasible_start(lo, warm_edges, alpha)
    for i, j in warm_edges:
        x[lo.off_z + edge_index(n, i, j)] = 1.0
    x[lo.off_nu:lo.off_nu + m] = np.maximum(0.0, x[lo.off_z:lo.off_z + m] - x[:m])
    d = np.zeros(pd.nx)
    y = x.copy()
    best_res, best_y, best_iter = math.inf, y.copy(), 0
    res, converged, ran = math.inf, False, 0
    trace = []
    for it in range(1, max_iter + 1):
        ran = it
        y = project_Y_het(pd, x, d)
        x, _ = update_X(pd, y, d)
        d += pd.rho * (x - y)
        res = float(np.sum((x - y) ** 2))
        trace.append((it, res, y[lo.lambda_ix], acf_of_g(n, y) if trace_acf else np.nan))
        if res < best_res:
            best_res, best_y, best_iter = res, y.copy(), it
        if res <= epsilon:
            converged = True
            break
    pick = y if converged else best_y
    note = "" if converged else f"stopped at max_iter; best iterate from iteration {best_iter}"
    sel = np.nonzero(pick[lo.off_z:lo.off_z + m] > 0.5)[0]
    weights = np.maximum(0.0, pick[:m])
    if len(sel) == 0:
        raise DegenerateSolutionError("no edge selected")
    if len(sel) < r:
        note = (note + "; " if note else "") + f"capacity limits stopped selection at {len(sel)} of {r} edges"
    e = enumerate_edges(n)
    node_sum = np.zeros(n)
    for l in sel:
        node_sum[e[l, 0]] += weights[l]
        node_sum[e[l, 1]] += weights[l]
    worst = node_sum.max()
    scale = 1.0 / worst if worst > 1.0 else 1.0
    edges, wts = e[sel], weights[sel] * scale
    w = gossip_matrix(n, edges, wts)
    rep = spectral_report(w)
    return Solution(edges, wts, w, rep["acf"], pick[lo.lambda_ix], converged, rep["connected"],
                    res if converged else best_res, ran, np.array(trace), note, False)
