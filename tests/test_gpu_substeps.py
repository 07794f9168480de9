"""GPU parity of the substeps through the C ABI against the oracle and the
reference goldens (proj/tests/test_admm.cpp, test_admm_het.cpp, test_eig.cpp,
test_bandwidth.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_X = 1e-9   # reference x-step is BiCGSTAB to 1e-13 here; ours is exact (FP64)
TOL_Y = 1e-11  # cone projections: FP64 sign iteration vs Householder/QL eigen-clamp


def test_substeps_vs_reference_goldens(T, golden):
    for c in golden("substeps.json"):
        x, d = np.array(c["x"]), np.array(c["d"])
        if c["kind"] == "hom":
            y = T.project_Y(c["n"], c["r"], x, d)
            xs, kkt = T.update_X(c["n"], c["r"], np.array(c["y"]), d)
        else:
            y = T.project_Y_het(c["degrees"], x, d)
            xs, kkt = T.update_X_het(c["degrees"], np.array(c["y"]), d)
        assert np.max(np.abs(y - np.array(c["y"]))) < TOL_Y
        assert np.max(np.abs(xs - np.array(c["xstep"]))) < TOL_X
        assert np.max(np.abs(kkt - np.array(c["kkt"]))) < 1e-6


@pytest.mark.parametrize("n,r", [(3, 2), (4, 3), (7, 9), (16, 32), (40, 100), (65, 300), (100, 400)])
def test_substeps_vs_oracle(T, O, n, r):
    rng = np.random.default_rng(n)
    pd = O.assemble(n, r, 2.0, 2.5)
    x = rng.standard_normal(pd.nx)
    d = rng.standard_normal(pd.nx) * 0.3
    y_o = O.project_Y(pd, x, d)
    y_g = T.project_Y(n, r, x, d, rho=2.5)
    assert np.max(np.abs(y_o - y_g)) < TOL_Y * max(1.0, np.abs(y_o).max())
    assert np.count_nonzero(y_g[:pd.m]) <= r
    x_o, kkt_o = O.update_X(pd, y_o, d)
    x_g, kkt_g = T.update_X(n, r, y_o, d, rho=2.5)
    assert np.max(np.abs(x_o - x_g)) < TOL_X
    # KKT rows: A x - 1e-8 mu = beq (proj/tests/test_admm.cpp:121-137)
    prod = pd.A @ x_g - 1e-8 * kkt_g[pd.nx:]
    assert np.max(np.abs(prod - pd.beq)) < 1e-6
    # stationarity: x + A^T mu = rhs
    rhs = O.kkt_rhs(pd, y_o, d)[:pd.nx]
    assert np.max(np.abs(x_g + pd.A.T @ kkt_g[pd.nx:] - rhs)) < 1e-8


def test_het_substeps_vs_oracle(T, O):
    rng = np.random.default_rng(11)
    for deg in ([2, 2, 2], [3, 3, 2, 2, 2, 2, 1, 1], [5] * 12, [9] * 32 + [3] * 32):
        pd = O.assemble_het_node(deg, 2.0, 1.0)
        x = rng.standard_normal(pd.nx)
        d = rng.standard_normal(pd.nx) * 0.1
        y_o = O.project_Y_het(pd, x, d)
        y_g = T.project_Y_het(deg, x, d)
        assert np.max(np.abs(y_o - y_g)) < TOL_Y * max(1.0, np.abs(y_o).max())
        x_o, kkt_o = O.update_X(pd, y_o, d)
        x_g, kkt_g = T.update_X_het(deg, y_o, d)
        # the stiff degree rows (1e8 DtD) make x accurate to ~1e-8 relative in
        # any FP64 method; the reference's own KKT residual target is 1e-10
        assert np.max(np.abs(x_o - x_g)) < 1e-7
        prod = pd.A @ x_g - 1e-8 * kkt_g[pd.nx:]
        assert np.max(np.abs(prod - pd.beq)) < 1e-6


def test_projection_semantics(T):
    # proj/tests/test_admm.cpp:36-77
    n, r = 3, 2
    lo = T.hom_layout(n)
    x = np.zeros(lo.nx)
    d = np.zeros(lo.nx)
    x[0], x[1], x[2], x[lo.lambda_ix] = 0.5, -0.2, 0.3, 0.8
    x[lo.off_s + 0], x[lo.off_s + 4], x[lo.off_s + 8] = 2.0, -3.0, 1.0
    x[lo.off_y + 0], x[lo.off_y + 1] = -1.0, 2.0
    x[lo.off_t + 0], x[lo.off_t + 4] = -1.0, 2.0
    y = T.project_Y(n, r, x, d)
    assert (y[0], y[1], y[2], y[lo.lambda_ix]) == (0.5, 0.0, 0.3, 0.8)
    assert abs(y[lo.off_s]) < 1e-12 and y[lo.off_s + 4] == pytest.approx(-3.0)
    assert abs(y[lo.off_s + 8]) < 1e-12
    assert (y[lo.off_y], y[lo.off_y + 1]) == (0.0, 2.0)
    assert abs(y[lo.off_t]) < 1e-12 and y[lo.off_t + 4] == pytest.approx(2.0)
    x[lo.lambda_ix] = -0.4
    assert T.project_Y(n, r, x, d)[lo.lambda_ix] == 0.0
    d[1] = 0.5
    assert T.project_Y(n, r, x, d)[1] == pytest.approx(0.3)


def test_top_r_ties_to_lower_index(T):
    # proj/tests/test_admm.cpp:79-99
    lo = T.hom_layout(4)
    x = np.zeros(lo.nx)
    x[:6] = [0.5, -0.2, 0.3, 0.4, 0.1, 0.2]
    y = T.project_Y(4, 3, x, np.zeros(lo.nx))
    assert y[:6].tolist() == [0.5, 0.0, 0.3, 0.4, 0.0, 0.0]
    lo = T.hom_layout(3)
    x = np.zeros(lo.nx)
    x[:3] = 0.4
    y = T.project_Y(3, 2, x, np.zeros(lo.nx))
    assert y[:3].tolist() == [0.4, 0.4, 0.0]


@pytest.mark.parametrize("n", [300, 400, 1024])
def test_top_r_large_with_ties(T, O, n):
    """keep_top_r with heavy ties: n=300 runs the one-CTA-per-solve select,
    n >= 362 (m >= 65536) the grid-wide select (select_kernels.cu)."""
    rng = np.random.default_rng(5 + n)
    lo = T.hom_layout(n)
    cases = [rng.choice([0.1, 0.2, 0.3, 0.25, -1.0], size=lo.m),            # heavy ties
             np.where(rng.random(lo.m) < 0.3, rng.random(lo.m), -rng.random(lo.m)),  # ties at 0 after the clamp
             np.round(rng.random(lo.m), 3),                                   # ~1000 tied values
             # one exponent for every value: the grid select's candidate
             # compaction overflows in every CTA (full-range rounds), with
             # ties and without
             0.5 + np.round(rng.random(lo.m), 4) / 2,
             0.5 + rng.random(lo.m) / 2,
             # 10 % of the values 1 + k 2^-40 (k < 64: the same top 44 bits),
             # the rest below 0.1: the rounds after the first run on the
             # compacted candidates down to the ties
             np.where(rng.random(lo.m) < 0.1, 1.0 + np.floor(rng.random(lo.m) * 64) * 2.0 ** -40,
                      rng.random(lo.m) * 0.1)]
    for vals in cases:
        x = np.zeros(lo.nx)
        x[:lo.m] = vals
        npos = int((vals > 0).sum())
        for r in sorted({1, 17, 1000, 5000, npos, npos + 3, lo.m - 1}):
            if not 1 <= r <= lo.m:
                continue
            y = T.project_Y(n, r, x, np.zeros(lo.nx))
            want = np.maximum(0.0, vals)
            O.keep_top_r(want, lo.m, r)
            assert np.array_equal(y[:lo.m], want), (n, r)


def test_binary_z(T):
    # proj/tests/test_admm_het.cpp:35-45
    assert T.project_binary_z([0.9, 0.1, 0.5], 2).tolist() == [1.0, 0.0, 1.0]
    assert T.project_binary_z([0.9, 0.1, 0.5], 3).tolist() == [1.0, 1.0, 1.0]
    assert T.project_binary_z([0.4, 0.4, 0.4], 1).tolist() == [1.0, 0.0, 0.0]
    assert T.project_binary_z([0.4, 0.4], 0).tolist() == [0.0, 0.0]
    assert T.project_binary_z([-0.0, 0.0, -1.0, 3.0], 2).tolist() == [1.0, 0.0, 0.0, 1.0]
    with pytest.raises(ValueError):
        T.project_binary_z([0.1], 2)


def test_binary_z_signed_random(T, O):
    rng = np.random.default_rng(3)
    v = np.round(rng.standard_normal(20000), 2)  # many ties, both signs
    for r in (0, 1, 10, 9999, 20000):
        assert np.array_equal(T.project_binary_z(v, r), O.project_binary_z(v, r))


def test_dual_update(T):
    # proj/tests/test_admm.cpp:139-144
    d = T.update_duals(np.ones(10), np.full(10, 0.25), np.full(10, 0.5), 2.5)
    assert np.allclose(d, 0.5 + 2.5 * 0.75)


def test_extraction(T):
    # proj/tests/test_admm.cpp:249-268
    e, w, W = T.extract_topology(3, 2, [0.9, 0.8, 1e-9], 1e-6)
    assert e.tolist() == [[0, 1], [0, 2]]
    assert w[0] == pytest.approx(0.9 / 1.7) and w[1] == pytest.approx(0.8 / 1.7)
    e, w, W = T.extract_topology(3, 1, [0.9, 0.8, 1e-9], 1e-6)
    assert e.tolist() == [[0, 1]] and w[0] == 0.9
    with pytest.raises(T.DegenerateSolutionError):
        T.extract_topology(3, 2, [0.0, 0.0, 0.0], 1e-6)
    with pytest.raises(ValueError):
        T.extract_topology(3, 0, [0.9, 0.8, 1e-9], 1e-6)


def test_extraction_vs_oracle(T, O):
    rng = np.random.default_rng(9)
    n = 50
    m = n * (n - 1) // 2
    g = np.where(rng.uniform(size=m) < 0.1, rng.uniform(0, 0.3, m), 0.0)
    for r in (5, 60, 200):
        e, w, _ = T.extract_topology(n, r, g, 1e-6)
        eo, wo, _ = O.extract_topology(n, r, g, 1e-6)
        assert e.tolist() == eo.tolist()
        assert np.array_equal(w, wo)  # same accumulation order -> bitwise


@pytest.mark.parametrize("n", [2, 3, 5, 16, 63, 64, 65, 128, 200, 256])
def test_cone_projections_vs_eigh(T, O, n):
    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((n, n))
    a = a + a.T
    p, q = T.project_psd(a), T.project_nsd(a)
    scale = np.linalg.norm(a)
    assert np.max(np.abs(p - O.project_psd(a))) < 1e-13 * scale
    assert np.max(np.abs(q - O.project_nsd(a))) < 1e-13 * scale
    assert np.max(np.abs(p + q - a)) < 1e-12 * scale  # Moreau (proj/tests/test_eig.cpp:118-122)
    assert np.array_equal(p, p.T) and np.array_equal(q, q.T)
    assert np.linalg.eigvalsh(p).min() >= -1e-12 * scale
    assert np.linalg.eigvalsh(q).max() <= 1e-12 * scale
    assert np.max(np.abs(T.project_psd(p) - p)) < 1e-12 * scale  # idempotent


def test_cone_clustered_spectrum(T, O):
    # eigenvalues spread over 16 decades around zero (the hard case for a sign iteration)
    rng = np.random.default_rng(1)
    n = 128
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.concatenate([np.logspace(-16, 1, n // 2), -np.logspace(-16, 1, n - n // 2)])
    a = (Q * ev) @ Q.T
    a = 0.5 * (a + a.T)
    # schedule bound (cone_kernels.cuh): 6.1e-13 of c = min(||A||_F, ||A||_inf)
    assert np.max(np.abs(T.project_psd(a) - O.project_psd(a))) < 1e-12 * np.linalg.norm(a)


def test_cone_fixed_points(T):
    # proj/tests/test_eig.cpp:126-130
    assert np.max(np.abs(T.project_psd(np.eye(5)) - np.eye(5))) < 1e-12
    assert np.linalg.norm(T.project_nsd(np.eye(5))) < 1e-12


def test_spectral_vs_reference(T, golden):
    for c in golden("spectral.json"):
        rep = T.spectral_edges(c["n"], c["edges"], c["weights"])
        assert rep["acf"] == pytest.approx(c["acf"], rel=1e-10, abs=1e-12)
        assert rep["lambda2"] == pytest.approx(c["lambda2"], rel=1e-10, abs=1e-12)
        assert rep["lambda_n"] == pytest.approx(c["lambda_n"], rel=1e-10, abs=1e-12)
        assert rep["connected"] == c["connected"]
        W = np.eye(c["n"])
        for (i, j), x in zip(c["edges"], c["weights"]):
            W[i, i] -= x
            W[j, j] -= x
            W[i, j] += x
            W[j, i] += x
        dense = T.spectral_report(W)
        assert dense["acf"] == pytest.approx(c["acf"], rel=1e-10, abs=1e-12)


def test_spectral_closed_forms(T):
    # exponential n=256: 7/9 ; ring: 1/3 + 2/3 cos(2 pi / n) (test_topology.cpp:160-165, 305-314)
    e, w = [], []
    n = 256
    from oracle.topoopt_oracle import generate_benchmark
    e, w = generate_benchmark("exponential", n)
    assert T.spectral_edges(n, e, w)["acf"] == pytest.approx(7 / 9, abs=1e-12)
    e, w = generate_benchmark("ring", n)
    assert T.spectral_edges(n, e, w)["acf"] == pytest.approx(1 / 3 + 2 / 3 * np.cos(2 * np.pi / n), abs=1e-12)


def test_spectral_disconnected(T):
    rep = T.spectral_edges(6, [[0, 1], [2, 3]], [0.3, 0.3])
    assert rep["lambda2"] == pytest.approx(1.0) and not rep["connected"]


def test_allocation_bit_exact(T, golden):
    for c in golden("allocation.json"):
        if c["status"] == 0:
            bu, e = T.allocate_edge_capacity(c["b"], c["r"], c["caps"])
            assert bu == c["b_unit"] and e.tolist() == c["e"]
        elif c["status"] == 2:
            with pytest.raises(T.InfeasibleError):
                T.allocate_edge_capacity(c["b"], c["r"], c["caps"])
        else:
            with pytest.raises(ValueError):
                T.allocate_edge_capacity(c["b"], c["r"], c["caps"])


def test_allocation_batch(T, golden):
    cases = [c for c in golden("allocation.json") if len(c["b"]) == 16 and c["caps"] is None]
    cases += [{"b": [9.76] * 8 + [3.25] * 8, "r": r} for r in range(8, 60)]
    b = np.array([c["b"] for c in cases])
    r = np.array([c["r"] for c in cases])
    bu, e, st = T.allocate_batch(b, r)
    for k, c in enumerate(cases):
        try:
            want = T.allocate_edge_capacity(c["b"], c["r"])
            assert st[k] == 0 and bu[k] == want[0] and e[k].tolist() == want[1].tolist()
        except T.InfeasibleError:
            assert st[k] == 2
