"""Quick diagnostics of the CUDA path against the oracle (run on a GPU box)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

try:
    from oracle import ref
    HAVE_REF = ref.available()
except Exception:  # pragma: no cover
    HAVE_REF = False


def step(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok]   {name} ({time.time() - t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def t_alloc():
    b = [9.76] * 8 + [3.25] * 8
    bu, e = T.allocate_edge_capacity(b, 16)
    bu2, e2 = O.allocate_edge_capacity(b, 16)
    print("  alloc", bu, e.tolist(), bu2 == bu, (e == e2).all())


def t_cone():
    rng = np.random.default_rng(0)
    for n in [3, 16, 64, 100, 256]:
        a = rng.standard_normal((n, n))
        a = a + a.T
        p = T.project_psd(a)
        q = T.project_nsd(a)
        e1 = np.abs(p - O.project_psd(a)).max()
        e2 = np.abs(q - O.project_nsd(a)).max()
        print(f"  cone n={n} psd err {e1:.2e} nsd err {e2:.2e} moreau {np.abs(p + q - a).max():.2e}")


def t_spec():
    rng = np.random.default_rng(1)
    for n in [2, 5, 16, 64, 200]:
        m = n * (n - 1) // 2
        g = np.zeros(m)
        idx = rng.choice(m, size=min(m, 3 * n), replace=False)
        g[idx] = rng.uniform(0, 1.0 / (3 * 3), len(idx))
        e = O.enumerate_edges(n)
        nz = g != 0
        w = O.gossip_matrix(n, e[nz], g[nz])
        a = O.spectral_report(w)
        b = T.spectral_report(w)
        c = T.spectral_edges(n, e[nz], g[nz])
        print(f"  spec n={n} oracle {a['acf']:.15f} dense {b['acf']:.15f} edges {c['acf']:.15f}"
              f" l2 {a['lambda2']:.6f}/{c['lambda2']:.6f}")


def t_substeps():
    rng = np.random.default_rng(2)
    for n, r in [(3, 2), (4, 3), (8, 10), (16, 32)]:
        pd = O.assemble(n, r, 2.0, 1.0)
        x = rng.standard_normal(pd.nx)
        d = rng.standard_normal(pd.nx) * 0.1
        y1 = O.project_Y(pd, x, d)
        y2 = T.project_Y(n, r, x, d)
        print(f"  project_Y n={n} max err {np.abs(y1 - y2).max():.2e}")
        xo, kkt = O.update_X(pd, y1, d)
        xg, kg = T.update_X(n, r, y1, d)
        print(f"  update_X n={n} max err {np.abs(xo - xg).max():.2e} mu err {np.abs(kkt - kg).max():.2e}")
    deg = [3, 3, 2, 2, 2, 2, 1, 1]
    pd = O.assemble_het_node(deg, 2.0, 1.0)
    x = rng.standard_normal(pd.nx)
    d = rng.standard_normal(pd.nx) * 0.1
    y1 = O.project_Y_het(pd, x, d)
    y2 = T.project_Y_het(deg, x, d)
    print(f"  project_Y_het max err {np.abs(y1 - y2).max():.2e}")
    xo, kkt = O.update_X(pd, y1, d)
    xg, kg = T.update_X_het(deg, y1, d)
    print(f"  update_X_het max err {np.abs(xo - xg).max():.2e} mu err {np.abs(kkt - kg).max():.2e}")


def t_solve16():
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=40000)
    t = time.time()
    s = T.solve(16, 32, **cfg)
    print(f"  solve16 {time.time() - t:.3f}s acf {s.acf_value!r} it {s.iterations} conv {s.converged}"
          f" edges {len(s.edges)} lam {s.lambda_tilde!r}")
    print("  first edges", s.edges[:6].tolist(), s.weights[:6].tolist())
    if HAVE_REF:
        r = ref.solve(16, 32, **cfg)
        print(f"  ref acf {r.acf!r} it {r.iterations} same edges {np.array_equal(r.edges, s.edges)}"
              f" max w rel {np.max(np.abs(r.weights - s.weights) / r.weights):.2e}")
        print(f"  trace acf max diff {np.nanmax(np.abs(r.trace[:, 3] - s.trace[:len(r.trace), 3])):.2e}")


def t_het():
    b = [9.76] * 32 + [3.25] * 32
    bu, e = T.allocate_edge_capacity(b, 192)
    cfg = dict(rho=10.0, epsilon=1e-8, max_iter=40000)
    t = time.time()
    s = T.solve_het(e, **cfg)
    print(f"  het64 {time.time() - t:.3f}s acf {s.acf_value!r} it {s.iterations} conv {s.converged}"
          f" edges {len(s.edges)} note {s.note!r}")


def t_big():
    for n, r in [(256, 1024), (1024, 4096)]:
        b = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=200)
        bu, e = T.allocate_edge_capacity([1.0] * n, r)
        warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1)
        b.set_warm(0, warm)
        b.start()
        b.iterate(8)
        b.sync()
        t = time.time()
        b.iterate(24)
        b.sync()
        dt = time.time() - t
        print(f"  n={n}: {24 / dt:.2f} iter/s ({dt / 24 * 1e3:.2f} ms/iter)")
        b.finish()
        s = b.result(0)
        print(f"    after {s.iterations} it residual {s.residual:.3e} acf {s.acf_value:.6f}"
              f" trace acf {s.trace[-3:, 3]}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["alloc", "cone", "spec", "substeps", "solve16", "het", "big"]
    for w in which:
        step(w, globals()["t_" + w])
