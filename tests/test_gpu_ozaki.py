"""GPU: the Ozaki-scheme FP64 GEMM on the int8 tensor cores (ozaki_kernels.cu)
against an exact numpy emulation of its digit-plane products, its digit-plane
output, determinism, and the cone projection against the FP64 DMMA path and
LAPACK."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KS = 7
_dp = C.POINTER(C.c_double)


def planes(M, e):
    """Balanced base-256 digits of rint(M 2^-e 2^(8 KS)) (what oz_split_kernel
    writes): digit s in [-128, 127], M = 2^e sum_s d_s 256^-s."""
    u = M * 2.0 ** (-e)
    assert np.abs(u).max() < 0.498
    q = np.rint(u * 2.0 ** (8 * KS)).astype(np.int64)
    Q = q + np.int64(int("80" * KS, 16))
    out = []
    for s in range(1, KS + 1):
        byte = (Q >> (8 * (KS - s))) & 0xFF
        out.append((byte - 128).astype(np.float64))
    return out


def emulate(A, eA, B, eB):
    """2^(eA+eB) sum_{d=KS+1..2} 2^-8d sum_{s+t=d} A_s B_t, lower tiles mirrored.
    Each A_s B_t is an exact integer matrix in float64 (|.| < 2^53)."""
    As, Bs = planes(A, eA), planes(B, eB)
    acc = np.zeros_like(A)
    for d in range(KS + 1, 1, -1):
        g = np.zeros_like(A)
        for s in range(max(1, d - KS), min(KS, d - 1) + 1):
            g += As[s - 1] @ Bs[d - s - 1]
        acc += g * 2.0 ** (-8 * d)
    acc *= 2.0 ** (eA + eB)
    return np.tril(acc) + np.tril(acc, -1).T


def sym(rng, n, bound):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M = (Q * rng.uniform(-bound, bound, n)) @ Q.T
    return 0.5 * (M + M.T)


def oz_gemm(lib, A, B, use_e=0, beta=0.0, digits=False, ec=3):
    nmat, ld, _ = A.shape
    Cg = np.zeros_like(A)
    Cd = np.zeros((nmat, KS, ld, ld), dtype=np.int8) if digits else None
    ms = C.c_double(0)
    rc = lib.tp_oz_gemm(ld, nmat, A.ctypes.data_as(_dp), 2, B.ctypes.data_as(_dp), 2, use_e, 1.0, beta,
                        Cg.ctypes.data_as(_dp), Cd.ctypes.data_as(C.c_void_p) if digits else None, ec, 0,
                        C.byref(ms))
    assert rc == 0, lib.tp_last_error_message()
    return Cg, Cd


@pytest.fixture(scope="module")
def lib():
    from paper_2512_07536_b200 import _lib
    return _lib.load()


@pytest.mark.parametrize("ld", [128, 256, 512])
def test_oz_gemm_equals_exact_emulation(lib, ld):
    rng = np.random.default_rng(ld)
    A = np.stack([sym(rng, ld, 1.2) for _ in range(2)])
    B = np.stack([sym(rng, ld, 1.4) for _ in range(2)])
    Cg, _ = oz_gemm(lib, A, B)
    for m in range(2):
        assert np.array_equal(Cg[m], emulate(A[m], 2, B[m], 2))  # bit for bit
        ex = A[m] @ B[m]
        ex = np.tril(ex) + np.tril(ex, -1).T
        assert np.max(np.abs(Cg[m] - ex)) < 1e-13 * np.abs(ex).max()
        assert np.array_equal(Cg[m], Cg[m].T)                     # exactly symmetric


def test_oz_gemm_epilogue_e_term(lib):
    rng = np.random.default_rng(7)
    A = np.stack([sym(rng, 256, 1.2) for _ in range(2)])
    B = np.stack([sym(rng, 256, 1.4) for _ in range(2)])
    Cg, _ = oz_gemm(lib, A, B, use_e=1, beta=0.5)
    for m in range(2):
        want = emulate(A[m], 2, B[m], 2) + 0.5 * A[m]
        assert np.max(np.abs(Cg[m] - want)) <= 4e-16 * np.abs(want).max()


def test_oz_digit_planes_output(lib):
    # the epilogue's digit planes reconstruct its own FP64 output to half a
    # unit of the last digit, 2^-(8 KS + 1) 2^e
    rng = np.random.default_rng(11)
    A = np.stack([sym(rng, 256, 1.2) for _ in range(2)])
    Cg, Cd = oz_gemm(lib, A, A, digits=True, ec=2)
    for m in range(2):
        rec = sum(Cd[m, s].astype(np.float64) * 2.0 ** (-8 * (s + 1)) for s in range(KS)) * 4.0
        assert np.max(np.abs(rec - Cg[m])) <= 2.0 ** -(8 * KS + 1) * 4.0
        assert np.array_equal(Cd[m], np.transpose(Cd[m], (0, 2, 1)))  # symmetric planes
        assert np.array_equal(Cd[m], np.stack(planes(Cg[m], 2)).astype(np.int8))  # rint digits


def test_oz_gemm_deterministic(lib):
    rng = np.random.default_rng(3)
    A = np.stack([sym(rng, 384, 1.2) for _ in range(2)])
    C1, D1 = oz_gemm(lib, A, A, digits=True)
    C2, D2 = oz_gemm(lib, A, A, digits=True)
    assert np.array_equal(C1, C2) and np.array_equal(D1, D2)


@pytest.mark.parametrize("n", [200, 384, 1000])
def test_cone_projection_vs_lapack(T, O, n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n))
    M = M + M.T
    M[: n // 3, : n // 3] *= 1e-6          # a cluster of small eigenvalues
    scale = np.linalg.norm(M)
    p_oz = T.project_psd(M)
    n_oz = T.project_nsd(M)
    assert np.max(np.abs(p_oz - O.project_psd(M))) < 1e-12 * scale
    assert np.max(np.abs(n_oz - O.project_nsd(M))) < 1e-12 * scale
    assert np.max(np.abs(p_oz - p_oz.T)) == 0.0
    # Moreau split (proj/tests/test_eig.cpp:89-124)
    assert np.max(np.abs(p_oz + n_oz - M)) < 1e-12 * scale
