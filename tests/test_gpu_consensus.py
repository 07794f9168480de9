"""GPU: consensus simulation (§8f row 2, proj/src/consensus.cpp:29-67) against
the compiled reference's traces, and the config-3 evaluation step (optimized
topology vs ring / exponential baselines)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_simulate_vs_reference(T, O, golden):
    for c in golden("consensus.json"):
        w = O.gossip_matrix(c["n"], np.array(c["edges"]), np.array(c["weights"]))
        err = T.simulate(w, c["dim"], c["iters"], c["seed"])
        ref = np.array(c["errors"])
        assert err[0] == ref[0]  # the reference's start state, bit for bit
        # the state evolves in the reference's arithmetic order; only the
        # per-step Frobenius sum is reassociated
        assert np.allclose(err, ref, rtol=1e-12, atol=0.0), c["label"]


def test_simulate_rejects_non_gossip(T):
    w = np.eye(4)
    w[0, 1] = 0.5
    with pytest.raises(ValueError):
        T.simulate(w, 2, 3, 0)
    with pytest.raises(ValueError):
        T.simulate(np.eye(3), 0, 3, 0)


def test_config3_vs_baselines(T, O, golden):
    # the optimized n=256, r=1024 topology against the
    # ring and exponential baselines (closed forms: proj/tests/test_topology.cpp)
    g = golden("config3.json")["solution"]
    w_opt = O.gossip_matrix(256, np.array(g["edges"]), np.array(g["weights"]))
    acf_opt = T.spectral_report(w_opt)["acf"]
    e, w = T.generate_benchmark("ring", 256)
    acf_ring = T.spectral_report(O.gossip_matrix(256, e, w))["acf"]
    e, w = T.generate_benchmark("exponential", 256)
    acf_exp = T.spectral_report(O.gossip_matrix(256, e, w))["acf"]
    assert acf_ring == pytest.approx(1 / 3 + 2 / 3 * np.cos(2 * np.pi / 256), rel=1e-10)
    assert acf_exp == pytest.approx(7 / 9, rel=1e-10)
    assert acf_opt == pytest.approx(g["acf"], rel=1e-6)
    assert acf_opt < acf_exp < acf_ring
    t_opt = T.convergence_time(T.simulate(w_opt, 16, 200, 0), 1e-6, 1.0)
    t_exp = T.convergence_time(T.simulate(O.gossip_matrix(256, e, w), 16, 200, 0), 1e-6, 1.0)
    assert t_opt < t_exp
