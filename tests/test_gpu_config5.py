"""GPU: config 5 (the batched n=256 sweep's node-level heterogeneous
scenarios) in lockstep with the compiled reference: the first 40 iterations
of the reference's solve_het loop (proj/src/admm_het.cpp:266-301) from the
sweep's warm start, two-tier and four-tier bandwidths at r=1024
(tests/golden/config5_lockstep.json, made by tests/golden/make_config5.py).
The reference's x-step is BiCGSTAB to 1e-10 relative, ours the exact
closed form, so the trajectories agree to the solve tolerance, not bitwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(rho=10.0, epsilon=1e-30)


def test_config5_lockstep_vs_reference(T, golden):
    g = golden("config5_lockstep.json")
    K = g["iterations"]
    for which, c in g["scenarios"].items():
        s = T.solve_het(np.array(c["degrees"]), warm_start=np.array(c["warm"]), max_iter=K, **CFG)
        assert s.iterations == K, which
        ref = np.array(c["trace"])           # residual, lambda, acf per iteration
        got = s.trace[:K, 1:4]
        rel_res = np.abs(got[:, 0] - ref[:, 0]) / ref[:, 0]
        assert rel_res.max() < 1e-5, (which, rel_res.max())
        assert np.abs(got[:, 1] - ref[:, 1]).max() < 1e-8, which       # lambda_tilde
        assert np.abs(got[:, 2] - ref[:, 2]).max() < 1e-6, which       # acf (trace SLEM tolerance)


def test_config5_batch_equals_single(T, golden):
    """Both scenarios in one lockstep batch (the sweep's layout) give the
    single solves' traces bit for bit."""
    g = golden("config5_lockstep.json")
    K = 12
    cases = list(g["scenarios"].values())
    singles = [T.solve_het(np.array(c["degrees"]), warm_start=np.array(c["warm"]), max_iter=K, **CFG)
               for c in cases]
    bs = T.BatchSolver(256, degrees=np.array([c["degrees"] for c in cases]), max_iter=K, **CFG)
    try:
        for b, c in enumerate(cases):
            bs.set_warm(b, np.array(c["warm"]))
        bs.start()
        bs.run()
        bs.finish()
        for b, one in enumerate(singles):
            got = bs.result(b)
            assert np.array_equal(got.trace, one.trace)
            assert got.edges.tolist() == one.edges.tolist()
    finally:
        bs.close()
