"""GPU: multi-iteration lockstep parity at the large configs (SURVEY §7/§8c:
the reference cannot finish an n=1024 solve, so n=1024 is pinned by lockstep
runs of the first k iterations from an explicit warm start).

The device solver and the numpy oracle (LAPACK eigen-clamps, exact top-r with
the reference's (value desc, index asc) rule, the closed-form KKT solve of
oracle.update_X_closed -- itself pinned to the sparse-LU KKT solve and to the
compiled reference) run the same k ADMM iterations (proj/src/admm.cpp:384-406)
independently from the same warm start. After every iteration: identical
top-r edge sets, Y/X/D within 1e-9 (relative to each block's max), and after
k iterations the trace rows (residual, lambda_tilde, acf_iterate) within
1e-6 relative. The top-r margin g_(r) - g_(r+1) is logged per iteration
(gpurun_out/lockstep_margins_n*.json) so that a flip would be diagnosable."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def warm_start(T, O, n, r):
    # the reference's annealer at steps=1, moves=1 on the
    # unit-bandwidth Alg. 1 allocation (run by the device annealer, which
    # reproduces the reference's draws: tests/test_gpu_anneal.py)
    bu, e = O.allocate_edge_capacity([1.0] * n, r)
    return np.asarray(T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)).reshape(-1, 2)


def block_rel(a, b, scale=None):
    den = max(np.abs(b).max() if scale is None else scale, 1e-300)
    return float(np.abs(a - b).max() / den)


BLOCKS = ("g", "lambda", "S", "y", "T")


def blocks(lo):
    n = lo.n
    return dict(zip(BLOCKS, ((0, lo.m), (lo.m, lo.m + 1), (lo.off_s, lo.off_s + n * n),
                             (lo.off_y, lo.off_y + n), (lo.off_t, lo.off_t + n * n))))


def check_blocks(lo, got, want, tol, what, it, scale_by=None, factor=1.0):
    """Per-block max error relative to the block's max |want| (or, for the
    duals D = D + rho (X - Y), a difference of nearly equal iterates, to
    factor * max |scale_by| of the block: errors in X and Y of e |X| move D
    by rho e |X|)."""
    for name, (s0, s1) in blocks(lo).items():
        sc = None if scale_by is None else factor * np.abs(scale_by[s0:s1]).max()
        e = block_rel(got[s0:s1], want[s0:s1], sc)
        assert e < tol, f"iteration {it}: {what}.{name} differs by {e:.3e} (relative)"


def top_r_margin(v, m, r):
    g = np.sort(np.maximum(0.0, v[:m]))[::-1]
    return float(g[r - 1] - g[r]) if r < m else float("inf")


@pytest.mark.parametrize("n,r,k", [(256, 1024, 12), (1024, 4096, 8)])
def test_lockstep_vs_oracle(T, O, n, r, k):
    rho, eps = 10.0, 1e-8
    warm = warm_start(T, O, n, r)
    pd = O.light_problem(n, r, 2.0, rho)
    lo = pd.lo
    bs = T.BatchSolver(n, r=[r], rho=rho, epsilon=eps, max_iter=k)
    margins = []
    try:
        bs.set_warm(0, warm)
        bs.start()
        X0 = bs.download()[0][0]
        x = O.feasible_start(lo, warm, 2.0)
        check_blocks(lo, X0, x, 1e-12, "X0", 0)
        d = np.zeros(lo.nx)
        rows = []
        for it in range(1, k + 1):
            margins.append(top_r_margin(x + d / rho, lo.m, r))
            y = O.project_Y(pd, x, d)
            x, _ = O.update_X_closed(pd, y, d)
            O.update_duals(pd, x, y, d)
            rows.append((float(np.sum((x - y) ** 2)), y[lo.lambda_ix], O.acf_of_g(n, y)))
            bs.iterate(1)
            bs.sync()
            Xg, Yg, Dg = (a[0] for a in bs.download())
            sel_g = np.nonzero(Yg[:lo.m] > 0)[0]
            sel_o = np.nonzero(y[:lo.m] > 0)[0]
            assert np.array_equal(sel_g, sel_o), f"iteration {it}: top-r edge sets differ"
            check_blocks(lo, Yg, y, 1e-9, "Y", it)
            check_blocks(lo, Xg, x, 1e-9, "X", it)
            check_blocks(lo, Dg, d, 1e-9, "D", it, scale_by=x, factor=rho)
        bs.finish()
        tr = bs.result(0).trace[:, 1:]  # (iter, residual, lambda_tilde, acf_iterate)
        want = np.array(rows)
        assert tr.shape[0] == k
        # residual = |X - Y|^2: its square root moves by at most the state error
        xnorm = float(np.linalg.norm(x))
        assert np.max(np.abs(np.sqrt(tr[:, 0]) - np.sqrt(want[:, 0]))) < 1e-9 * xnorm
        for c in (1, 2):  # lambda_tilde, acf_iterate: 1e-6 relative (north star)
            rel = np.abs(tr[:, c] - want[:, c]) / np.maximum(np.abs(want[:, c]), 1e-300)
            assert rel.max() < 1e-6, (c, rel)
    finally:
        bs.close()
        out = os.path.join(ROOT, "gpurun_out")
        if os.path.isdir(out):
            with open(os.path.join(out, f"lockstep_margins_n{n}.json"), "w") as f:
                json.dump({"n": n, "r": r, "iterations": len(margins), "top_r_margin": margins}, f)
    assert min(margins) > 0.0


@pytest.mark.slow
def test_n1024_one_iteration_vs_compiled_reference(T, O):
    """One ADMM iteration at n=1024 against the compiled reference's own
    substeps (oracle/_ref): its feasible start, project_Y (Householder + QL
    eigen-clamps) and update_X (ILU(0) BiCGSTAB, restarted every 10 steps as
    SURVEY §8d sanctions, to 1e-10). ~1 minute of reference CPU time."""
    from oracle import ref
    if not ref.available():
        pytest.skip("compiled reference (oracle/_ref) not built")
    n, r, rho = 1024, 4096, 10.0
    warm = warm_start(T, O, n, r)
    rp = ref.Problem(n, r, 2.0, rho)
    x0 = rp.feasible_start(warm)
    d = np.zeros(rp.nx)
    y_ref = rp.project_Y(x0, d)
    kkt = np.zeros(rp.nx + rp.neq)
    x_ref = rp.update_X(y_ref, d, kkt, tol=1e-10, chunk=10)
    bs = T.BatchSolver(n, r=[r], rho=rho, epsilon=1e-8, max_iter=1)
    try:
        bs.set_warm(0, warm)
        bs.start()
        lo = O.light_problem(n, r, 2.0, rho).lo
        check_blocks(lo, bs.download()[0][0], x0, 1e-12, "X0", 0)
        bs.iterate(1)
        bs.sync()
        Xg, Yg, _ = (a[0] for a in bs.download())
    finally:
        bs.close()
    assert np.array_equal(np.nonzero(Yg[:lo.m] > 0)[0], np.nonzero(y_ref[:lo.m] > 0)[0])
    check_blocks(lo, Yg, y_ref, 1e-9, "Y", 1)
    # the reference's BiCGSTAB stops at 1e-10 relative residual
    check_blocks(lo, Xg, x_ref, 1e-7, "X", 1)
