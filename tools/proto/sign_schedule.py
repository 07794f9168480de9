"""Prototype of the FP64 polynomial sign iteration used for the PSD/NSD
projection. Checks accuracy against LAPACK eigh."""
import numpy as np, sys, time

QUINTIC = (3.4445, -4.7750, 2.0315)

def proj_psd_poly(A, k1=24, k2=6, sym=True):
    f = np.linalg.norm(A)
    if f == 0: return np.zeros_like(A), 0
    X = A / f
    a, b, c = QUINTIC
    ng = 0
    for _ in range(k1):
        Y = X @ X
        Z = c * (Y @ Y) + b * Y
        X = X @ Z + a * X
        ng += 3
        if sym: X = np.tril(X) + np.tril(X, -1).T
    for _ in range(k2):
        Y = X @ X
        X = -0.5 * (X @ Y) + 1.5 * X
        ng += 2
        if sym: X = np.tril(X) + np.tril(X, -1).T
    P = 0.5 * (A @ X) + 0.5 * A
    ng += 1
    P = np.tril(P) + np.tril(P, -1).T
    return P, ng

def proj_psd_eig(A):
    w, V = np.linalg.eigh(0.5*(A+A.T))
    return (V * np.maximum(w, 0)) @ V.T

rng = np.random.default_rng(0)
for n in [16, 64, 256, 1024]:
    for kind in ["gauss", "lowrank_pos", "clustered"]:
        if kind == "gauss":
            A = rng.standard_normal((n, n)); A = A + A.T
        else:
            Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
            if kind == "lowrank_pos":
                ev = -np.abs(rng.standard_normal(n)) * 10
                k = max(1, n // 10)
                ev[:k] = np.abs(rng.standard_normal(k)) * 1e-3
                ev[k:k+3] = [1e-12, -1e-12, 0.0]
            else:
                ev = np.concatenate([np.logspace(-16, 1, n//2), -np.logspace(-16, 1, n - n//2)])
            A = (Q * ev) @ Q.T; A = 0.5 * (A + A.T)
        t = time.time()
        for k1 in ([20, 24] if n <= 256 else [24]):
            P, ng = proj_psd_poly(A, k1=k1)
            E = proj_psd_eig(A)
            err = np.linalg.norm(P - E) / np.linalg.norm(A)
            print(f"n={n:5d} {kind:12s} k1={k1} gemms={ng} relerr={err:.2e}  maxabs={np.abs(P-E).max():.2e}")


# ---------------------------------------------------------------------------
# Schedule design for the Ozaki path (cone_kernels.cuh: ozaki_schedule()).
# band_quintic(kappa, U): LP over odd quintics p(x) = x (a + b x^2 + c x^4)
# maximising the guaranteed growth g = min_{x in (0, kappa]} p(x)/x while
# keeping p([0, U]) <= U and p([kappa, U]) >= kappa (the band is invariant).
# scalar_error(steps): the projection error bound max_mu mu |1 - s(mu)| / 2
# (relative to ||A||_F) of a schedule, from the scalar map on a log grid.
# (0.55, 1.3) with 20 steps + 6 Newton-Schulz: 73 products, 4.4e-14;
# the Muon quintic needs 22 + 6 = 79 products for 1.8e-14 and 21 + 6 = 76
# for 6.3e-14.
def band_quintic(kappa, U, n=1500):
    from scipy.optimize import linprog
    x1 = np.linspace(1e-9, kappa, n); x2 = np.linspace(0, U, n); x3 = np.linspace(kappa, U, n)
    rows = [[-1, -x * x, -x ** 4, 1] for x in x1] + [[x, x ** 3, x ** 5, 0] for x in x2] + \
           [[-x, -x ** 3, -x ** 5, 0] for x in x3]
    rhs = [0] * n + [U] * n + [-kappa] * n
    r = linprog([0, 0, 0, -1], A_ub=np.array(rows), b_ub=np.array(rhs), bounds=[(None, None)] * 4,
                method="highs")
    return tuple(r.x[:3]), r.x[3]


def scalar_error(quintic, k1, k2):
    mu = np.concatenate([np.geomspace(1e-17, 1, 200000), np.linspace(0.5, 1, 20001)])
    a, b, c = quintic
    x = mu.copy()
    for _ in range(k1):
        x = x * (a + b * x * x + c * x ** 4)
    for _ in range(k2):
        x = 1.5 * x - 0.5 * x ** 3
    return (mu * np.abs(1 - x) / 2).max(), 3 * k1 + 2 * k2 + 1
