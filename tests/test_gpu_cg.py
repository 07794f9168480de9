"""GPU: the CG linear substep (linear_solver = 1) against
the closed-form x-step, the oracle's sparse-LU KKT solve and the reference
goldens. The reference's update_X is BiCGSTAB + ILU(0) to linear_tol on the
full KKT system (proj/src/admm.cpp:279-293, proj/src/solvers.cpp:109-227);
ours is matrix-free CG on the g block of the same delta-regularised system."""
import numpy as np
import pytest

from test_gpu_solve import check_against

pytestmark = pytest.mark.gpu

TOL_X = 1e-9


@pytest.mark.parametrize("n,r", [(3, 2), (16, 32), (65, 300), (256, 1024), (1024, 4096)])
def test_update_X_cg_vs_closed_form_and_oracle(T, O, n, r):
    rng = np.random.default_rng(100 + n)
    pd = O.assemble(n, r, 2.0, 2.5)
    y = rng.standard_normal(pd.nx)
    d = rng.standard_normal(pd.nx) * 0.3
    x_c, kkt_c = T.update_X(n, r, y, d, rho=2.5)
    x_g, kkt_g, its, rel = T.update_X_cg(n, r, y, d, rho=2.5, linear_tol=1e-10)
    # H_gg has three eigenvalues on the complete graph: CG stops after <= 3
    assert 1 <= its <= 3 and rel <= 1e-10
    assert np.max(np.abs(x_g - x_c)) < 1e-11 * max(1.0, np.abs(x_c).max())
    assert np.max(np.abs(kkt_g - kkt_c)) < 1e-6
    if n <= 65:
        x_o, _ = O.update_X(pd, y, d)
        assert np.max(np.abs(x_o - x_g)) < TOL_X


def test_update_X_cg_reference_goldens(T, golden):
    for c in golden("substeps.json"):
        if c["kind"] != "hom":
            continue
        xs, _, its, rel = T.update_X_cg(c["n"], c["r"], np.array(c["y"]), np.array(c["d"]))
        assert np.max(np.abs(xs - np.array(c["xstep"]))) < TOL_X
        assert rel <= 1e-10


def test_update_X_cg_guard_and_zero_rhs(T, O):
    n, r = 16, 32
    lo = T.hom_layout(n)
    # one CG iteration cannot reach 1e-8 on a generic right-hand side: the
    # reference's LinearSolveError (proj/src/admm.cpp:287)
    rng = np.random.default_rng(3)
    y = rng.standard_normal(lo.nx)
    d = rng.standard_normal(lo.nx)
    with pytest.raises(T.LinearSolveError):
        T.update_X_cg(n, r, y, d, cg_max_iter=1)
    # a right-hand side with h = 0 on the edges is solved in zero iterations
    pd = O.assemble(n, r, 2.0, 1.0)
    x0 = np.zeros(lo.nx)
    xs, _ = T.update_X(n, r, x0, x0)
    xc, _, its, rel = T.update_X_cg(n, r, x0, x0)
    assert np.max(np.abs(xs - xc)) < 1e-13
    assert pd.nx == lo.nx


def test_config1_golden_with_cg(T, golden):
    g = golden("config1.json")
    s = T.solve(16, 32, warm_start=g["warm"], linear_solver=1, **g["cfg"])
    check_against(s, g["solution"])


def test_small_solves_golden_with_cg(T, golden):
    for c in golden("small_solves.json"):
        if c["kind"] != "hom":
            continue
        s = T.solve(c["n"], c["r"], warm_start=c["warm"], linear_solver=1, **c["cfg"])
        check_against(s, c["solution"])


def test_cg_rejects_het(T):
    with pytest.raises(ValueError):
        T.solve_het([2, 2, 2, 2], linear_solver=1)
    with pytest.raises(ValueError):
        T.SolverConfig(linear_solver=2).validate()


def test_n1024_lockstep_cg_vs_closed_form(T, O):
    n, r = 1024, 4096
    bu, e = O.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=6)
    a = T.solve(n, r, warm_start=warm, **cfg)
    b = T.solve(n, r, warm_start=warm, linear_solver=1, **cfg)
    assert a.iterations == b.iterations == 6
    ta, tb = a.trace, b.trace
    # residuals sum (x - y)^2 of small differences (|x - y| ~ 1e-3): CG's
    # 1e-10 relative solve tolerance moves them by ~1e-7 relative; the
    # north-star tolerance (1e-6 relative) is the bar
    assert np.max(np.abs(ta[:, 1] - tb[:, 1]) / np.abs(ta[:, 1])) < 1e-6
    assert np.max(np.abs(ta[:, 2] - tb[:, 2])) < 1e-10                     # lambda_tilde
    assert a.edges.tolist() == b.edges.tolist()
    assert np.max(np.abs(a.weights - b.weights)) < 1e-9
    sv = T.BatchSolver(n, r=[r], linear_solver=1, **cfg)
    try:
        sv.set_warm(0, warm)
        sv.start()
        sv.iterate(2)
        sv.sync()
        its, rel = sv.cg_stats(0)
        assert 1 <= its <= 3 and rel <= 1e-10
    finally:
        sv.close()


@pytest.mark.parametrize("n,r,B", [(16, 32, 600), (65, 300, 100), (1024, 4096, 2)])
def test_cg_batched_global_equals_single_register(T, n, r, B):
    """A single solve's CG x-step runs the register-resident kernel (each of
    its tiles fits one co-resident CTA); a batch too large for that runs the
    global-memory kernel. Same arithmetic and reduction order, so every solve
    of the batch equals the single solve bit for bit (state trace, edges,
    weights)."""
    bu_e = T.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(bu_e[1], steps=1, moves_per_temp=1, seed=0)
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=4, linear_solver=1)
    one = T.solve(n, r, warm_start=warm, **cfg)
    bs = T.BatchSolver(n, r=[r] * B, **cfg)
    try:
        for b in range(B):
            bs.set_warm(b, warm)
        bs.start()
        bs.run()
        bs.finish()
        for b in sorted({0, B // 2, B - 1}):
            got = bs.result(b)
            assert np.array_equal(got.trace, one.trace)
            assert got.edges.tolist() == one.edges.tolist()
            assert np.array_equal(got.weights, one.weights)
            assert got.acf_value == one.acf_value  # the final report (8-CTA cluster per solve)
    finally:
        bs.close()


def test_solve_raises_linear_solve_error_like_the_reference(T):
    """update_X throws LinearSolveError when the linear solve misses 1e-8
    relative (proj/src/admm.cpp:287); solve() propagates it. One CG
    iteration per x-step cannot reach it on a generic iterate."""
    with pytest.raises(T.LinearSolveError):
        T.solve(16, 32, linear_solver=1, cg_max_iter=1, max_iter=50)
