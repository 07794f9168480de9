"""Generate the golden fixtures from the compiled reference (oracle/_ref).

Run in the development container (it needs /root/reference to build
oracle/_ref): ``make -C oracle && python tests/golden/make_golden.py``.
Every fixture records the reference's own outputs for the inputs stored next
to them; the GPU box only reads the committed JSON files.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DESIGN = dict(rho=10.0, epsilon=1e-8)


def sol_dict(s, trace=True):
    d = {"edges": s.edges.tolist(), "weights": s.weights.tolist(), "acf": s.acf,
         "lambda_tilde": s.lambda_tilde, "residual": s.residual, "converged": s.converged,
         "connected": s.connected, "repaired": s.repaired, "iterations": s.iterations,
         "note": s.note}
    if trace:
        d["trace"] = s.trace.tolist()
    return d


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name)


def config1():
    warm = ref.default_warm_start(16, 32, 0)
    s = ref.solve(16, 32, max_iter=40000, **DESIGN)
    dump("config1.json", {"n": 16, "r": 32, "cfg": {**DESIGN, "max_iter": 40000},
                          "warm": warm.tolist(), "solution": sol_dict(s)})


def config2():
    b = [9.76] * 32 + [3.25] * 32
    bu, e = ref.allocate(b, 192)
    warm = ref.anneal_degree(e, seed=0)
    s = ref.solve_het_node(e, warm_edges=warm, max_iter=40000, **DESIGN)
    dump("config2.json", {"bandwidths": b, "r": 192, "b_unit": bu, "degrees": e.tolist(),
                          "cfg": {**DESIGN, "max_iter": 40000}, "warm": warm.tolist(),
                          "solution": sol_dict(s)})


def small_cases():
    cases = []
    # proj/tests/test_admm.cpp:146-247 and acceptance-style settings
    for (n, r, cfg, warm) in [
        (2, 1, {"max_iter": 5000}, None),
        (4, 6, {"max_iter": 8000}, None),
        (3, 3, {**DESIGN, "max_iter": 10000}, None),
        (5, 6, {**DESIGN, "max_iter": 10000}, None),
        (6, 9, {**DESIGN, "max_iter": 10000}, None),
        (5, 6, {"max_iter": 2000}, None),
        (4, 6, {"max_iter": 3}, None),
        (3, 3, {"epsilon": 1e30}, None),
        (5, 4, {**DESIGN, "max_iter": 10000}, [[0, 1], [0, 2], [0, 3], [0, 4]]),
        (8, 12, {**DESIGN, "max_iter": 40000}, None),
        (12, 24, {**DESIGN, "max_iter": 40000}, None),
    ]:
        w = ref.default_warm_start(n, r, 0) if warm is None else np.array(warm)
        s = ref.solve(n, r, warm_edges=w, **cfg)
        cases.append({"kind": "hom", "n": n, "r": r, "cfg": cfg, "warm": np.asarray(w).tolist(),
                      "solution": sol_dict(s)})
    for deg in ([2, 2, 2], [3, 3, 2, 2, 2, 2, 1, 1], [2, 2, 2, 1, 1], [3] * 8 + [1] * 8,
                [6] * 8 + [2] * 8):
        warm = ref.anneal_degree(deg, seed=0)
        cfg = {**DESIGN, "max_iter": 3000}
        s = ref.solve_het_node(deg, warm_edges=warm, **cfg)
        cases.append({"kind": "het", "degrees": list(deg), "cfg": cfg, "warm": warm.tolist(),
                      "solution": sol_dict(s)})
    dump("small_solves.json", cases)


def substeps():
    rng = np.random.default_rng(2024)
    out = []
    for n, r in [(3, 2), (3, 3), (4, 3), (8, 10), (16, 32), (24, 60)]:
        p = ref.Problem(n, r, 2.0, 1.0)
        x = rng.standard_normal(p.nx)
        d = rng.standard_normal(p.nx) * 0.1
        y = p.project_Y(x, d)
        warm = np.zeros(p.nx + p.neq)
        xs = p.update_X(y, d, warm, tol=1e-13)
        out.append({"kind": "hom", "n": n, "r": r, "x": x.tolist(), "d": d.tolist(),
                    "y": y.tolist(), "xstep": xs.tolist(), "kkt": warm.tolist()})
    for deg in ([2, 2, 2], [3, 3, 2, 2, 2, 2, 1, 1], [4] * 10):
        p = ref.Problem(len(deg), degrees=deg, alpha=2.0, rho=1.0)
        x = rng.standard_normal(p.nx)
        d = rng.standard_normal(p.nx) * 0.1
        y = p.project_Y(x, d)
        warm = np.zeros(p.nx + p.neq)
        xs = p.update_X(y, d, warm, tol=1e-13, chunk=50)
        out.append({"kind": "het", "degrees": deg, "x": x.tolist(), "d": d.tolist(),
                    "y": y.tolist(), "xstep": xs.tolist(), "kkt": warm.tolist()})
    dump("substeps.json", out)


def allocation():
    rng = np.random.default_rng(51)
    cases = []
    for trial in range(300):
        n = 2 + int(rng.integers(31))
        b = ((1 + rng.integers(1280, size=n)) / 64.0).tolist()
        caps = rng.integers(n, size=n).tolist() if rng.uniform() < 0.5 else None
        r = 1 + int(rng.integers(n * (n - 1) // 2))
        try:
            bu, e = ref.allocate(b, r, caps)
            cases.append({"b": b, "caps": caps, "r": r, "status": 0, "b_unit": bu, "e": e.tolist()})
        except ref.RefError as exc:
            cases.append({"b": b, "caps": caps, "r": r, "status": exc.status})
    # the two-tier goldens of proj/tests/test_bandwidth.cpp:38-52 and config 2/5 profiles
    for b, r in [([9.76] * 8 + [3.25] * 8, 16), ([9.76] * 8 + [3.25] * 8, 32),
                 ([9.76] * 32 + [3.25] * 32, 192), ([1.0] * 4, 6), ([1.0] * 1024, 4096),
                 ([9.76] * 128 + [3.25] * 128, 1024),
                 ([9.76] * 64 + [6.5] * 64 + [4.88] * 64 + [3.25] * 64, 800)]:
        bu, e = ref.allocate(b, r)
        cases.append({"b": b, "caps": None, "r": r, "status": 0, "b_unit": bu, "e": e.tolist()})
    dump("allocation.json", cases)


def warm_starts():
    cases = []
    for n, r, seed in [(16, 32, 0), (6, 8, 5), (8, 12, 0), (12, 24, 3), (64, 192, 0), (5, 3, 0)]:
        cases.append({"kind": "default", "n": n, "r": r, "seed": seed,
                      "edges": ref.default_warm_start(n, r, seed).tolist()})
    for deg, steps, moves, seed in [([8] * 256, 1, 1, 0), ([8] * 1024, 1, 1, 0),
                                    ([3, 3, 2, 2, 2, 2, 1, 1], 200, 0, 0)]:
        cases.append({"kind": "anneal", "degrees": deg, "steps": steps, "moves": moves, "seed": seed,
                      "edges": ref.anneal_degree(deg, steps=steps, moves_per_temp=moves,
                                                 seed=seed).tolist()})
    dump("warm_starts.json", cases)


def spectral():
    cases = []
    for kind in ("ring", "exponential"):
        for n in (4, 8, 16, 64, 128, 256):
            e, w = ref.generate_benchmark(kind, n)
            W = np.eye(n)
            for (i, j), x in zip(e, w):
                W[i, i] -= x
                W[j, j] -= x
                W[i, j] += x
                W[j, i] += x
            rep = ref.spectral_report(W)
            cases.append({"kind": kind, "n": n, "edges": e.tolist(), "weights": w.tolist(), **rep})
    dump("spectral.json", cases)


if __name__ == "__main__":
    which = sys.argv[1:] or ["config1", "small_cases", "substeps", "allocation", "warm_starts",
                             "spectral", "config2"]
    for w in which:
        globals()[w]()
