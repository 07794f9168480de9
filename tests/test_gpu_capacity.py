"""GPU: capacity-bound heterogeneous systems (§8f row 3): the capped binary
projection, the capacity annealer and solve_het on intra-server tree and
BCube rows, against the compiled reference (tests/golden/capacity.json;
proj/tests/test_admm_het.cpp:47-229, acceptance.cpp:238-268)."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def system(T, spec):
    return T.tiered8_tree_system(*spec[1:]) if spec[0] == "tiered8" else T.bcube_constraints(*spec[1:])


def test_capped_projection(T, golden):
    for c in golden("capacity.json")["capped"]:
        z = T.project_binary_z_capped(np.array(c["v"]), c["r"], system(T, c["spec"]))
        assert z.tolist() == c["z"]


def test_capacity_anneal(T, golden):
    for c in golden("capacity.json")["anneal"]:
        e = T.anneal_capacity_topology(system(T, c["spec"]), c["r"], steps=c["steps"], seed=c["seed"])
        assert e.tolist() == c["edges"]


def test_capacity_solves(T, golden):
    for c in golden("capacity.json")["solves"]:
        sys_ = system(T, c["spec"])
        if c["drop_last"]:
            sys_.rows.pop()
            sys_.capacities.pop()
        s = T.solve_het_capacity(sys_, c["r"], warm_start=np.array(c["warm"]), **c["cfg"])
        ref = c["solution"]
        assert s.iterations == ref["iterations"]
        assert s.converged == ref["converged"]
        assert s.edges.tolist() == ref["edges"]
        assert rel(s.weights, ref["weights"]) < 1e-6
        assert s.acf_value == pytest.approx(ref["acf"], rel=1e-6, abs=1e-9)
        assert s.connected == ref["connected"]
        assert s.note == ref["note"]
        tr = np.array(ref["trace"])
        assert np.max(np.abs(s.trace[:, 3] - tr[:, 3])) < 1e-6
        # every capacity row holds and only allowed pairs appear
        n = sys_.n
        sel = np.zeros(n * (n - 1) // 2, np.int8)
        for i, j in s.edges:
            sel[i * n - i * (i + 1) // 2 + (j - i - 1)] = 1
        assert all(ld <= cap for ld, cap in zip(sys_.loads(sel), sys_.capacities))
        assert all(sys_.allowed[k] for k in np.nonzero(sel)[0])


def test_capacity_default_warm_start(T):
    # no warm start: anneal_topology on the system (proj/src/anneal.cpp:393-407)
    sys_ = T.tiered8_tree_system()
    s = T.solve_het_capacity(sys_, 12, rho=10.0, epsilon=1e-8, max_iter=3000)
    assert s.connected and len(s.edges) <= 12
