"""GPU end-to-end parity of solve / solve_het against the reference goldens
(config 1 golden, config 2 golden, proj/tests/test_admm.cpp and
test_admm_het.cpp behaviours). Edge sets must be identical; weights and SLEM
within 1e-6 relative (FP64)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel

pytestmark = pytest.mark.gpu


def check_against(s, ref, wtol=1e-6):
    assert s.iterations == ref["iterations"]
    assert s.converged == ref["converged"]
    assert s.edges.tolist() == ref["edges"]
    assert rel(s.weights, ref["weights"]) < wtol
    assert s.acf_value == pytest.approx(ref["acf"], rel=1e-6, abs=1e-9)
    assert s.lambda_tilde == pytest.approx(ref["lambda_tilde"], rel=1e-6, abs=1e-9)
    assert s.connected == ref["connected"]
    tr = np.array(ref["trace"])
    assert s.trace.shape == tr.shape
    assert np.max(np.abs(s.trace[:, 2] - tr[:, 2])) < 1e-6          # lambda_tilde
    assert np.max(np.abs(s.trace[:, 3] - tr[:, 3])) < 1e-6          # acf_iterate


def test_config1_golden(T, golden):
    g = golden("config1.json")
    s = T.solve(16, 32, warm_start=g["warm"], **g["cfg"])
    check_against(s, g["solution"])
    assert s.acf_value <= 0.57  # acceptance gate 2 (proj/tests/acceptance.cpp:83-96)


def test_config1_default_warm_start(T, golden):
    # no warm start passed: the host annealer must reproduce the reference's
    g = golden("config1.json")
    s = T.solve(16, 32, **g["cfg"])
    check_against(s, g["solution"])


def test_default_warm_starts(T, golden):
    for c in golden("warm_starts.json"):
        if c["kind"] == "default":
            assert T.default_warm_start(c["n"], c["r"], c["seed"]).tolist() == c["edges"]


def test_small_solves_golden(T, golden):
    for c in golden("small_solves.json"):
        if c["kind"] == "hom":
            s = T.solve(c["n"], c["r"], warm_start=c["warm"], **c["cfg"])
        else:
            s = T.solve_het(c["degrees"], warm_start=c["warm"], **c["cfg"])
        check_against(s, c["solution"])
        assert s.note == c["solution"]["note"]
        assert s.repaired == c["solution"]["repaired"]


def test_config2_het_golden(T, golden):
    if not os.path.exists(os.path.join(GOLDEN, "config2.json")):
        pytest.skip("config2 fixture missing")
    g = golden("config2.json")
    bu, e = T.allocate_edge_capacity(g["bandwidths"], g["r"])
    assert bu == g["b_unit"] and e.tolist() == g["degrees"]
    s = T.solve_het(e, warm_start=g["warm"], **g["cfg"])
    check_against(s, g["solution"])
    assert s.edges.shape[0] == g["r"]


def test_two_node_and_full_support(T):
    # proj/tests/test_admm.cpp:146-168
    s = T.solve(2, 1, max_iter=5000)
    assert s.converged and s.connected and s.acf_value < 1e-3
    assert s.weights[0] == pytest.approx(0.5, rel=1e-3)
    s = T.solve(4, 6, max_iter=8000)
    assert s.converged and s.connected and s.acf_value <= 0.02 and len(s.edges) == 6
    assert np.allclose(s.weights, 0.25, rtol=0.05) and s.lambda_tilde > 0.9


def test_invariants(T, O):
    # proj/tests/test_admm.cpp:170-193
    for n, r in [(3, 3), (5, 6), (6, 9)]:
        s = T.solve(n, r, rho=10.0, epsilon=1e-8, max_iter=10000)
        assert s.converged and s.residual <= 1e-8 and len(s.edges) <= r
        w = O.gossip_matrix(n, s.edges, s.weights)
        assert np.max(np.abs(w - s.w)) < 1e-12
        assert s.acf_value == pytest.approx(O.spectral_report(w)["acf"], rel=1e-10)
        assert s.acf_value <= 1.0 - s.lambda_tilde + 0.05
        assert s.trace[-1, 1] == pytest.approx(s.residual)


def test_bitwise_reproducible(T):
    # proj/tests/test_admm.cpp:195-207 (and deterministic reductions on the GPU)
    a = T.solve(5, 6, max_iter=2000)
    b = T.solve(5, 6, max_iter=2000)
    assert a.iterations == b.iterations and a.residual == b.residual
    assert a.edges.tolist() == b.edges.tolist() and np.array_equal(a.weights, b.weights)
    assert np.array_equal(a.trace, b.trace, equal_nan=True)
    h1 = T.solve_het([2, 2, 2, 1, 1], rho=10.0, epsilon=1e-8, max_iter=3000)
    h2 = T.solve_het([2, 2, 2, 1, 1], rho=10.0, epsilon=1e-8, max_iter=3000)
    assert h1.edges.tolist() == h2.edges.tolist() and h1.acf_value == h2.acf_value


def test_iteration_cap_and_trace_csv(T):
    # proj/tests/test_admm.cpp:209-229
    s = T.solve(4, 6, max_iter=3)
    assert not s.converged and s.iterations == 3 and s.note and len(s.trace) == 3
    assert s.trace_csv().startswith("iter,residual,lambda_tilde,acf_iterate\n")
    s = T.solve(3, 3, epsilon=1e30)
    assert s.converged and s.iterations >= 1


def test_warm_start_validation(T):
    with pytest.raises(ValueError):
        T.solve(4, 2, warm_start=[[0, 1], [1, 2], [2, 3]])
    with pytest.raises(ValueError):
        T.solve(4, 3, warm_start=[[0, 5]])
    with pytest.raises(ValueError):
        T.solve_het([1, 1, 2], warm_start=[[0, 1], [0, 2], [1, 2]])
    with pytest.raises(T.InfeasibleError):
        T.solve_het([1, 1, 1])


def test_exponential_dominance(T, O):
    # acceptance gate 3 (proj/tests/acceptance.cpp:100-119)
    for n in (8, 12, 16):
        e, w = O.generate_benchmark("exponential", n)
        exp_acf = O.spectral_report(O.gossip_matrix(n, e, w))["acf"]
        s = T.solve(n, len(e), rho=10.0, epsilon=1e-8, max_iter=40000)
        assert s.connected and s.acf_value <= exp_acf + 0.01


def test_config3_golden(T, golden):
    # n=256, r=1024, the reference's default warm start
    if not os.path.exists(os.path.join(GOLDEN, "config3.json")):
        pytest.skip("config3 fixture missing")
    g = golden("config3.json")
    ref = g["solution"]
    assert T.default_warm_start(g["n"], g["r"], 0).tolist() == g["warm"]
    s = T.solve(g["n"], g["r"], warm_start=g["warm"], **g["cfg"])
    assert s.converged == ref["converged"]
    assert s.edges.tolist() == ref["edges"]
    assert rel(s.weights, ref["weights"]) < 1e-6
    assert s.acf_value == pytest.approx(ref["acf"], rel=1e-6)
    assert s.lambda_tilde == pytest.approx(ref["lambda_tilde"], rel=1e-6)
    assert s.connected == ref["connected"]
    # the iteration count depends on when ||X - Y||^2 crosses 1e-8: within 1 %
    assert abs(s.iterations - ref["iterations"]) <= 0.01 * ref["iterations"]
    rows = [i for i in ref["trace_rows"] if i < s.trace.shape[0]]
    tr = np.array(ref["trace"])[: len(rows)]
    assert np.max(np.abs(s.trace[rows, 2] - tr[:, 2])) < 1e-6   # lambda_tilde
    assert np.max(np.abs(s.trace[rows, 3] - tr[:, 3])) < 1e-6   # acf_iterate


def test_solve_plan_cache_bitwise(T, golden):
    """tp_solve reuses the thread's last solver plan (buffers + graphs) for the
    same shape: a reused plan, with another warm start and another shape in
    between, returns bitwise what a fresh solver returns."""
    n, r = 64, 150
    bu, e = T.allocate_edge_capacity([1.0] * n, r)
    w0 = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
    w1 = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=1)
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=300)
    T.release_solver_plans()
    fresh = T.solve(n, r, warm_start=w0, **cfg)
    T.solve(n, r, warm_start=w1, **cfg)           # same plan, other state
    again = T.solve(n, r, warm_start=w0, **cfg)
    T.solve(16, 32, warm_start=golden("config1.json")["warm"], rho=10.0, epsilon=1e-8)  # evicts
    third = T.solve(n, r, warm_start=w0, **cfg)
    for s in (again, third):
        assert s.iterations == fresh.iterations and s.converged == fresh.converged
        assert np.array_equal(s.trace, fresh.trace)
        assert s.edges.tolist() == fresh.edges.tolist() and np.array_equal(s.weights, fresh.weights)
        assert s.acf_value == fresh.acf_value
    T.release_solver_plans()
