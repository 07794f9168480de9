"""Accuracy study: the polynomial sign-iteration projection with every GEMM
done as an exact integer (int8-slice) product, Ozaki scheme I with a fixed
per-operand power-of-two scale taken from a static spectral bound.

  M ~= 2^e * sum_{s=1..k} 2^{-7s} M_s,   M_s int8 in [-127, 127] (truncated digits)
  A.B ~= 2^{eA+eB} sum_{s+t <= k+1} 2^{-7(s+t)} (A_s . B_t)       (exact int32 products)

numpy float64 matmuls of the slices are exact (|sum| < 2^53), so this emulates
the tcgen05 kind::i8 kernel bit for bit up to the FP64 epilogue order.
Usage: python tools/proto/ozaki.py [n ...]
"""
import sys
import time

import numpy as np

QA, QB, QC = 3.4445, -4.7750, 2.0315


def slices(M, e, k):
    u = M * 2.0 ** (-e)
    assert np.abs(u).max() < 1.0, (np.abs(u).max(), e)
    out = []
    for _ in range(k):
        u = u * 128.0
        d = np.trunc(u)
        out.append(d)
        u = u - d
    return out


def ozaki_mm(Asl, eA, Bsl, eB, k, order="desc"):
    acc = np.zeros_like(Asl[0])
    # group by d = s + t, smallest contributions first
    for d in range(k + 1, 1, -1):
        g = np.zeros_like(Asl[0])
        for s in range(1, d):
            t = d - s
            if s <= k and t <= k:
                g += Asl[s - 1] @ Bsl[t - 1]
        acc += g * 2.0 ** (-7 * d)
    acc = acc * 2.0 ** (eA + eB)
    return np.tril(acc) + np.tril(acc, -1).T   # lower tiles computed, mirrored


def sym(M):
    return np.tril(M) + np.tril(M, -1).T


def proj_psd(A, k, k1=22, k2=6, exact=False):
    f = np.linalg.norm(A)
    X = A / f

    def mm(P, eP, Q, eQ):
        if exact:
            return sym(P @ Q)
        return ozaki_mm(slices(P, eP, k), eP, slices(Q, eQ, k), eQ, k)

    eX0 = 1
    for it in range(k1):
        Y = mm(X, 1, X, 1)
        Z = QC * mm(Y, 1, Y, 1) + QB * Y
        X = mm(X, 1, Z, 2) + QA * X
    for it in range(k2):
        Y = mm(X, 1, X, 1)
        X = -0.5 * mm(X, 1, Y, 1) + 1.5 * X
    X0 = A / f
    P = 0.5 * f * (mm(X0, eX0, X, 1) + X0)
    return 0.5 * (P + P.T)


def proj_eig(A):
    w, V = np.linalg.eigh(0.5 * (A + A.T))
    return (V * np.maximum(w, 0)) @ V.T


KS = (7, 8, 9)


def main():
    ns = [int(a) for a in sys.argv[1:]] or [64, 256]
    rng = np.random.default_rng(0)
    for n in ns:
        for kind in ["gauss", "lowrank_pos", "clustered"]:
            if kind == "gauss":
                A = rng.standard_normal((n, n))
                A = A + A.T
            else:
                Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
                if kind == "lowrank_pos":
                    ev = -np.abs(rng.standard_normal(n)) * 10
                    r = max(1, n // 10)
                    ev[:r] = np.abs(rng.standard_normal(r)) * 1e-3
                    ev[r:r + 3] = [1e-12, -1e-12, 0.0]
                else:
                    ev = np.concatenate([np.logspace(-16, 1, n // 2), -np.logspace(-16, 1, n - n // 2)])
                A = (Q * ev) @ Q.T
                A = 0.5 * (A + A.T)
            E = proj_eig(A)
            fa = np.linalg.norm(A)
            t = time.time()
            P = proj_psd(A, 0, exact=True)
            print(f"n={n:5d} {kind:12s} fp64      relerr={np.linalg.norm(P - E) / fa:.2e}", flush=True)
            for k in KS:
                P = proj_psd(A, k)
                print(f"n={n:5d} {kind:12s} ozaki k={k} pairs={k * (k + 1) // 2:2d} "
                      f"relerr={np.linalg.norm(P - E) / fa:.2e} maxabs/fa={np.abs(P - E).max() / fa:.2e}"
                      f"  ({time.time() - t:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
