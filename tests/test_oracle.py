"""CPU: the numpy oracle (oracle/topoopt_oracle.py) pinned against the
reference's golden fixtures (tests/golden/, generated from the compiled
reference by tests/golden/make_golden.py) and, when oracle/_ref is built,
against the reference itself."""
import numpy as np
import pytest

from conftest import rel


def test_layout_dimensions(O):
    # proj/tests/test_admm.cpp:15-34 and test_admm_het.cpp:80-108
    lo = O.hom_layout(2)
    assert (lo.m, lo.nx, lo.neq) == (1, 12, 10)
    lo = O.hom_layout(16)
    assert (lo.m, lo.nx, lo.neq) == (120, 649, 528)
    assert O.hom_layout(4).nx + O.hom_layout(4).neq == 43 + 36
    het = O.het_layout(3, 3)
    assert (het.nx, het.neq) == (31, 27)
    pd = O.assemble_het_node([2, 2, 2])
    assert list(pd.beq[21:24]) == [2.0, 2.0, 2.0] and list(pd.beq[24:27]) == [0.0, 0.0, 0.0]
    with pytest.raises(ValueError):
        O.assemble(4, 0)
    with pytest.raises(ValueError):
        O.assemble(4, 7)


def test_edge_index_roundtrip(O):
    for n in (2, 3, 7, 64):
        e = O.enumerate_edges(n)
        for l, (i, j) in enumerate(e):
            assert O.edge_index(n, i, j) == l == O.edge_index(n, j, i)


def test_allocation_bit_exact_vs_reference(O, golden):
    for c in golden("allocation.json"):
        if c["status"] == 0:
            bu, e = O.allocate_edge_capacity(c["b"], c["r"], c["caps"])
            assert bu == c["b_unit"]  # bitwise
            assert e.tolist() == c["e"]
        elif c["status"] == 2:
            with pytest.raises(O.InfeasibleError):
                O.allocate_edge_capacity(c["b"], c["r"], c["caps"])
        else:
            with pytest.raises(ValueError):
                O.allocate_edge_capacity(c["b"], c["r"], c["caps"])


def test_two_tier_allocation_goldens(O):
    # proj/tests/test_bandwidth.cpp:38-52
    b = [9.76] * 8 + [3.25] * 8
    bu, e = O.allocate_edge_capacity(b, 16)
    assert bu == pytest.approx(3.25) and e.tolist() == [3] * 8 + [1] * 8
    bu, e = O.allocate_edge_capacity(b, 32)
    assert bu == pytest.approx(1.625) and e.tolist() == [6] * 8 + [2] * 8


def test_substeps_vs_reference(O, golden):
    for c in golden("substeps.json"):
        if c["kind"] == "hom":
            pd = O.assemble(c["n"], c["r"], 2.0, 1.0)
            y = O.project_Y(pd, np.array(c["x"]), np.array(c["d"]))
        else:
            pd = O.assemble_het_node(c["degrees"], 2.0, 1.0)
            y = O.project_Y_het(pd, np.array(c["x"]), np.array(c["d"]))
        assert np.max(np.abs(y - np.array(c["y"]))) < 1e-12
        x, kkt = O.update_X(pd, np.array(c["y"]), np.array(c["d"]))
        # the reference solves to 1e-13 relative with BiCGSTAB; same system
        assert np.max(np.abs(x - np.array(c["xstep"]))) < 1e-9


def test_spectral_vs_reference(O, golden):
    for c in golden("spectral.json"):
        W = O.gossip_matrix(c["n"], c["edges"], c["weights"])
        rep = O.spectral_report(W)
        assert rep["acf"] == pytest.approx(c["acf"], rel=1e-12, abs=1e-14)
        assert rep["lambda2"] == pytest.approx(c["lambda2"], rel=1e-12, abs=1e-14)
        assert rep["connected"] == c["connected"]


def test_exponential_closed_form(O):
    # proj/tests/test_topology.cpp:305-314: exponential graph ACF (m-1)/(m+1)
    e, w = O.generate_benchmark("exponential", 256)
    rep = O.spectral_report(O.gossip_matrix(256, e, w))
    assert rep["acf"] == pytest.approx(7.0 / 9.0, abs=1e-12)


def test_config1_full_solve_vs_reference(O, golden):
    g = golden("config1.json")
    s = O.solve(16, 32, g["warm"], **g["cfg"])
    ref = g["solution"]
    assert s.iterations == ref["iterations"] and s.converged
    assert s.edges.tolist() == ref["edges"]
    assert rel(s.weights, ref["weights"]) < 1e-6
    assert s.acf == pytest.approx(ref["acf"], rel=1e-9)
    tr = np.array(ref["trace"])
    assert np.max(np.abs(s.trace[:, 3] - tr[:, 3])) < 1e-6


def test_small_solves_vs_reference(O, golden):
    for c in golden("small_solves.json"):
        ref = c["solution"]
        if c["kind"] == "hom":
            s = O.solve(c["n"], c["r"], c["warm"], **c["cfg"])
        else:
            s = O.solve_het_node(c["degrees"], c["warm"], **c["cfg"])
        assert s.iterations == ref["iterations"], c
        assert s.converged == ref["converged"]
        assert s.edges.tolist() == ref["edges"]
        assert np.max(np.abs(s.weights - np.array(ref["weights"]))) < 1e-6
        assert s.acf == pytest.approx(ref["acf"], rel=1e-6, abs=1e-9)


@pytest.mark.slow
def test_config2_het_vs_reference(O, golden):
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, "config2.json")):
        pytest.skip("config2 fixture not generated")
    g = golden("config2.json")
    s = O.solve_het_node(g["degrees"], g["warm"], **g["cfg"])
    ref = g["solution"]
    assert s.iterations == ref["iterations"]
    assert s.edges.tolist() == ref["edges"]
    assert s.acf == pytest.approx(ref["acf"], rel=1e-6)


def test_oracle_against_live_reference():
    from oracle import ref, topoopt_oracle as O
    if not ref.available():
        pytest.skip("oracle/_ref not built (run make -C oracle)")
    rng = np.random.default_rng(7)
    for n, r in [(5, 4), (7, 9), (10, 20)]:
        p = ref.Problem(n, r, 2.0, 3.0)
        pd = O.assemble(n, r, 2.0, 3.0)
        x = rng.standard_normal(p.nx)
        d = rng.standard_normal(p.nx)
        assert np.max(np.abs(p.project_Y(x, d) - O.project_Y(pd, x, d))) < 1e-12
        assert np.array_equal(p.beq, pd.beq)
        fs = p.feasible_start(ref.default_warm_start(n, r, 1))
        fo = O.feasible_start(pd.lo, ref.default_warm_start(n, r, 1), 2.0)
        assert np.max(np.abs(fs - fo)) < 1e-12


def test_consensus_simulate_vs_golden(O, golden):
    # proj/src/consensus.cpp:29-67 against the compiled reference
    for c in golden("consensus.json"):
        if c["n"] > 64:
            continue  # the n=256 cases are checked on the GPU
        w = O.gossip_matrix(c["n"], np.array(c["edges"]), np.array(c["weights"]))
        err = O.simulate(w, c["dim"], c["iters"], c["seed"])
        ref = np.array(c["errors"])
        assert np.allclose(err, ref, rtol=1e-10, atol=1e-13 * ref[0])


def test_generate_benchmark_python_mirror(T, golden):
    # the Python mirror of generate_benchmark against the reference's graphs
    for c in golden("spectral.json"):
        if c["kind"] in ("ring", "grid2d", "torus2d", "exponential"):
            e, w = T.generate_benchmark(c["kind"], c["n"])
            assert e.tolist() == c["edges"]
            assert np.array_equal(w, np.array(c["weights"]))


def _capsys(c):
    rows = [c["cols"][c["row_ptr"][k]:c["row_ptr"][k + 1]] for k in range(len(c["caps"]))]
    return rows, c["caps"], c["allowed"]


def test_capacity_system_builders(T, golden):
    # intra_server_constraints(tiered8_tree) / bcube_constraints vs the reference
    g = golden("capacity.json")["systems"]
    built = {"tiered8": T.tiered8_tree_system(4.88, 4.88, 9.76), "bcube_4_2": T.bcube_constraints(4, 2),
             "bcube_2_2": T.bcube_constraints(2, 2), "bcube_3_2": T.bcube_constraints(3, 2),
             "bcube_3_1": T.bcube_constraints(3, 1)}
    for name, sys_ in built.items():
        ptr, cols, caps, al = sys_.csr()
        c = g[name]
        assert ptr.tolist() == c["row_ptr"] and cols[: len(c["cols"])].tolist() == c["cols"]
        assert caps[: len(c["caps"])].tolist() == c["caps"] and al.tolist() == c["allowed"]


def test_capped_projection_oracle(O, golden):
    g = golden("capacity.json")
    name = lambda s: "tiered8" if s[0] == "tiered8" else f"bcube_{s[1]}_{s[2]}"  # noqa: E731
    for c in g["capped"]:
        z = O.project_binary_z_capped(np.array(c["v"]), c["r"], *_capsys(g["systems"][name(c["spec"])]))
        assert z.tolist() == c["z"]


def test_capacity_solve_oracle(O, golden):
    g = golden("capacity.json")
    name = lambda s: "tiered8" if s[0] == "tiered8" else f"bcube_{s[1]}_{s[2]}"  # noqa: E731
    for c in g["solves"][:3]:
        rows, caps, al = _capsys(g["systems"][name(c["spec"])])
        n = g["systems"][name(c["spec"])]["n"]
        s = O.solve_het_capacity(n, rows, caps, al, c["r"], c["warm"], trace_acf=False, **c["cfg"])
        ref = c["solution"]
        assert s.iterations == ref["iterations"] and s.edges.tolist() == ref["edges"]
        assert rel(s.weights, ref["weights"]) < 1e-6
        assert s.acf == pytest.approx(ref["acf"], rel=1e-6) and s.note == ref["note"]


def test_formats_vs_reference(T, golden):
    # §8f row 4: topology.json / w.csv / trace.csv against the reference's own
    # serializers (proj/src/topology.cpp:283-324, admm.cpp:223-236), byte for
    # byte (the oracle's nlohmann prints as stock 3.11.3, oracle/Makefile)
    for c in golden("formats.json"):
        ours = T.topology_to_json(c["n"], c["edges"], c["weights"])
        assert ours == c["topology_json"], c["label"]
        w = T.gossip_matrix(c["n"], np.array(c["edges"]), np.array(c["weights"]))
        assert T.matrix_to_csv(w) == c["w_csv"]
        if "trace_csv" in c:
            rows = [r.split(",") for r in c["trace_csv"].strip().split("\n")[1:]]
            tr = np.array([[float(x) for x in r] for r in rows])
            assert T.trace_csv(tr) == c["trace_csv"]
        n, e, wt = T.topology_from_json(ours)
        e0, w0 = T.normalize_topology(c["n"], c["edges"], c["weights"])
        assert n == c["n"] and np.array_equal(e, e0) and np.array_equal(wt, w0)


def test_json_number_format(T):
    # nlohmann::json double layout (shortest round trip, fixed for exponents in (-5, 15])
    cases = {0.5: "0.5", 1.0: "1.0", 100.0: "100.0", 1e-05: "1e-05", 0.0001: "0.0001",
             2.0 ** -20: "9.5367431640625e-07", 0.30000000000000004: "0.30000000000000004",
             1e15: "1e+15", 123456789012345.0: "123456789012345.0", -2.5: "-2.5", 0.0: "0.0",
             1.5e300: "1.5e+300"}
    for v, s in cases.items():
        assert T.json_number(v) == s, (v, T.json_number(v))


def test_write_optimize_artifacts(T, golden, tmp_path):
    """The optimize command's files (proj/tools/topoopt.cpp:244-296) byte for
    byte against the reference's serializers and the CLI's own json objects."""
    c = golden("formats.json")[0]
    rows = [r.split(",") for r in c["trace_csv"].strip().split("\n")[1:]]
    tr = np.array([[float(x) for x in r] for r in rows])
    e, w = np.array(c["edges"]), np.array(c["weights"])
    sv = c["solution"]
    sol = T.Solution(e, w, T.gossip_matrix(16, e, w), sv["lambda_tilde"], sv["acf"], sv["converged"],
                     sv["connected"], sv["repaired"], sv["residual"], sv["iterations"], sv["note"], tr)
    al = c["allocation"]
    files = T.write_optimize_artifacts(str(tmp_path), "homogeneous", sol, warm=e,
                                       allocation=(al["b_unit"], al["e"]))
    assert files == ["allocation.json", "solution.json", "topology.json", "trace.csv", "w.csv",
                     "warm_start.json"]
    assert (tmp_path / "topology.json").read_text() == c["topology_json"]
    assert (tmp_path / "w.csv").read_text() == c["w_csv"]
    assert (tmp_path / "trace.csv").read_text() == c["trace_csv"]
    assert (tmp_path / "solution.json").read_text() == c["solution_json"]
    assert (tmp_path / "allocation.json").read_text() == c["allocation_json"]


@pytest.mark.parametrize("n", [3, 5, 16, 33])
def test_closed_form_xstep_equals_kkt_lu(O, n):
    """oracle.update_X_closed (the slack-eliminated KKT solve used for the
    n=1024 lockstep parity) equals the sparse-LU solve of the assembled
    delta-regularised KKT (proj/src/admm.cpp:46-94, 279-293)."""
    rng = np.random.default_rng(100 + n)
    pd = O.assemble(n, n, 2.0, 2.5)
    y = rng.standard_normal(pd.nx)
    d = rng.standard_normal(pd.nx) * 0.3
    x1, k1 = O.update_X(pd, y, d)
    x2, k2 = O.update_X_closed(O.light_problem(n, n, 2.0, 2.5), y, d)
    assert np.abs(x1 - x2).max() < 1e-13 * np.abs(x1).max()
    assert np.abs(k1 - k2).max() < 1e-13 * np.abs(k1).max()
