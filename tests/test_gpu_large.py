"""GPU: large-n parity through size-independent properties (the reference
cannot finish n=1024 solves), lockstep substeps at n=1024 against
LAPACK, and batched/sharded solves against single solves (bitwise)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def feasible_state(T, O, n, r, seed):
    bu, e = O.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=seed)
    lo = O.hom_layout(n)
    return O.feasible_start(lo, warm, 2.0), warm


@pytest.mark.parametrize("n,r", [(256, 1024), (1024, 4096)])
def test_project_Y_large_vs_lapack(T, O, n, r):
    rng = np.random.default_rng(n)
    x, _ = feasible_state(T, O, n, r, 0)
    lo = O.hom_layout(n)
    d = np.zeros(lo.nx)
    # perturb so the cones have both signs and the top-r has competition
    x[:lo.m] += rng.standard_normal(lo.m) * 1e-3
    s = rng.standard_normal((n, n)) * 1e-2
    x[lo.off_s:lo.off_s + n * n] += (s + s.T).reshape(-1)
    t = rng.standard_normal((n, n)) * 1e-2
    x[lo.off_t:lo.off_t + n * n] += (t + t.T + np.diag(rng.standard_normal(n)) * 1e-2).reshape(-1)
    y = T.project_Y(n, r, x, d, rho=10.0)
    # edges: clamp + exact top-r with the reference tie rule
    want = np.maximum(0.0, x[:lo.m])
    O.keep_top_r(want, lo.m, r)
    assert np.array_equal(y[:lo.m], want)
    # cones against LAPACK
    S = x[lo.off_s:lo.off_s + n * n].reshape(n, n).T
    Tm = x[lo.off_t:lo.off_t + n * n].reshape(n, n).T
    ys = y[lo.off_s:lo.off_s + n * n].reshape(n, n).T
    yt = y[lo.off_t:lo.off_t + n * n].reshape(n, n).T
    assert np.max(np.abs(ys - O.project_nsd(S))) < 1e-12 * np.linalg.norm(S)
    assert np.max(np.abs(yt - O.project_psd(Tm))) < 1e-12 * np.linalg.norm(Tm)


@pytest.mark.parametrize("n,r", [(256, 1024), (1024, 4096)])
def test_update_X_large_kkt_properties(T, O, n, r):
    rng = np.random.default_rng(n + 1)
    x, _ = feasible_state(T, O, n, r, 1)
    lo = O.hom_layout(n)
    y = x + rng.standard_normal(lo.nx) * 1e-2
    d = rng.standard_normal(lo.nx) * 1e-2
    xs, kkt = T.update_X(n, r, y, d, rho=10.0)
    pd = O.assemble(n, r, 2.0, 10.0)
    mu = kkt[lo.nx:]
    rhs = y - d / 10.0
    rhs[lo.lambda_ix] += 1.0 / 10.0
    # the two block rows of [[I, A^T], [A, -1e-8 I]] [x; mu] = [rhs; beq]
    assert np.max(np.abs(xs + pd.A.T @ mu - rhs)) < 1e-9
    assert np.max(np.abs(pd.A @ xs - 1e-8 * mu - pd.beq)) < 1e-9


def test_batched_equals_single(T):
    n, rs = 16, [32, 24, 40, 20]
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=40000)
    bs = T.BatchSolver(n, r=rs, **cfg)
    warms = [T.default_warm_start(n, r, 0) for r in rs]
    for b, w in enumerate(warms):
        bs.set_warm(b, w)
    bs.start()
    bs.run()
    bs.finish()
    for b, r in enumerate(rs):
        got = bs.result(b)
        one = T.solve(n, r, warm_start=warms[b], **cfg)
        assert got.iterations == one.iterations
        assert got.edges.tolist() == one.edges.tolist()
        assert np.array_equal(got.weights, one.weights)
        assert got.acf_value == one.acf_value


def test_batched_oneoff_reports_equal_single(T):
    """n = 400: the one-off SLEM reports (feasible start, final) run the plain
    Lanczos recurrence as an 8-CTA cluster per solve, the incidence from
    global memory in a batch and from shared memory alone; both give the
    single solve's report bit for bit, for every solve of the batch."""
    n, rs = 400, [1200, 1000, 1400]
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=6)
    warms = [T.default_warm_start(n, r, 0) for r in rs]
    bs = T.BatchSolver(n, r=rs, **cfg)
    try:
        for b, w in enumerate(warms):
            bs.set_warm(b, w)
        bs.start()
        bs.run()
        bs.finish()
        for b, r in enumerate(rs):
            got = bs.result(b)
            one = T.solve(n, r, warm_start=warms[b], **cfg)
            assert 0.0 < got.acf_value < 1.0
            assert got.acf_value == one.acf_value
            assert np.array_equal(got.trace, one.trace)
            assert got.edges.tolist() == one.edges.tolist()
    finally:
        bs.close()


def test_batched_het_equals_single(T):
    n = 16
    degs = [[3] * 8 + [1] * 8, [6] * 8 + [2] * 8, [4] * 16]
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=3000)
    bs = T.BatchSolver(n, degrees=degs, **cfg)
    warms = [T.anneal_degree_topology(d) for d in degs]
    for b, w in enumerate(warms):
        bs.set_warm(b, w)
    bs.start()
    bs.run()
    bs.finish()
    for b, d in enumerate(degs):
        got = bs.result(b)
        one = T.solve_het(d, warm_start=warms[b], **cfg)
        assert got.iterations == one.iterations
        assert got.edges.tolist() == one.edges.tolist()
        assert np.array_equal(got.weights, one.weights)


def test_n1024_iterations_run_and_decrease(T):
    n, r = 1024, 4096
    bu, e = T.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1)
    bs = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=40)
    bs.set_warm(0, warm)
    bs.start()
    bs.iterate(40)
    assert bs.sync()
    bs.finish()
    s = bs.result(0)
    assert s.iterations == 40 and not s.converged
    assert np.all(np.isfinite(s.trace[:, 1])) and np.all(np.isfinite(s.trace[:, 3]))
    assert s.trace[-1, 1] < s.trace[0, 1]
    assert len(s.edges) <= r and s.connected
