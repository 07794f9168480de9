"""CPU: the C-ABI library builds, loads and exports every symbol declared in
include/topoopt_b200.h; compute entry points fail loudly without a GPU (no CPU
fallback). The host-side warm-start annealer matches the reference bit for
bit (it runs on the host, no device needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "topoopt_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tp_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2512_07536_b200 import _lib
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"


def test_config_defaults_match_reference():
    # SolverConfig defaults, proj/include/topoopt/admm.hpp:15-25
    from paper_2512_07536_b200 import _lib
    c = _lib.tp_config()
    _lib.load().tp_config_default(C.byref(c))
    assert (c.rho, c.epsilon, c.max_iter, c.alpha, c.weight_floor, c.seed, c.linear_tol) == \
        (1.0, 1e-6, 20000, 2.0, 1e-6, 0, 1e-10)
    assert _lib.load().tp_config_validate(C.byref(c)) == 0


@pytest.mark.parametrize("field,value", [("epsilon", 0.0), ("max_iter", 0), ("alpha", -2.0),
                                         ("weight_floor", -1e-9), ("linear_tol", 0.0), ("rho", -1.0)])
def test_config_validation(T, field, value):
    # proj/tests/test_admm.cpp:297-313
    cfg = T.SolverConfig(**{field: value})
    with pytest.raises(ValueError):
        cfg.validate()


def test_no_cpu_fallback(T):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(T.CudaError):
        T.project_psd(np.eye(3))
    with pytest.raises(T.CudaError):
        T.solve(4, 3)


def test_host_annealer_matches_reference(T, golden):
    for c in golden("warm_starts.json"):
        if c["kind"] != "anneal":
            continue
        e = T.anneal_degree_topology(c["degrees"], steps=c["steps"], moves_per_temp=c["moves"],
                                     seed=c["seed"])
        assert e.tolist() == c["edges"]


def test_host_annealer_infeasible(T):
    with pytest.raises(T.InfeasibleError):
        T.anneal_degree_topology([1, 1, 1])  # odd degree sum
    with pytest.raises(T.InfeasibleError):
        T.anneal_degree_topology([2, 2, 0, 0])  # zero degree
    with pytest.raises(ValueError):
        T.anneal_degree_topology([5, 1, 1, 1])  # degree >= n


def test_edge_index_and_layout(T):
    assert T.edge_index(16, 0, 5) == 4
    assert T.edge_index(16, 5, 0) == 4
    lo = T.het_layout(3, 3)
    assert (lo.nx, lo.neq) == (31, 27)
    with pytest.raises(ValueError):
        T.edge_index(4, 2, 2)
