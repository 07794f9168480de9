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
