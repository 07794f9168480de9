"""GPU: the Ozaki-scheme FP64 GEMM on the int8 tensor cores (ozaki_kernels.cu)
against an exact numpy emulation of its digit-plane products, its digit-plane
output, determinism, and the cone projection against the FP64 DMMA path and
LAPACK."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KS = 8
_dp = C.POINTER(C.c_double)


def planes(M, e):
    """Truncated base-128 digits of M 2^-e (what oz_split_kernel writes)."""
    u = M * 2.0 ** (-e)
    assert np.abs(u).max() < 1.0
    out = []
    for _ in range(KS):
        u = u * 128.0
        d = np.trunc(u)
        out.append(d)
        u = u - d
    return out


def emulate(A, eA, B, eB):
    """2^(eA+eB) sum_{d=9..2} 2^-7d sum_{s+t=d} A_s B_t, lower tiles mirrored.
    Each A_s B_t is an exact integer matrix in float64 (|.| < 2^53)."""
    As, Bs = planes(A, eA), planes(B, eB)
    acc = np.zeros_like(A)
    for d in range(KS + 1, 1, -1):
        g = np.zeros_like(A)
        for s in range(max(1, d - KS), min(KS, d - 1) + 1):
            g += As[s - 1] @ Bs[d - s - 1]
        acc += g * 2.0 ** (-7 * d)
    acc *= 2.0 ** (eA + eB)
    return np.tril(acc) + np.tril(acc, -1).T


def sym(rng, n, bound):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M = (Q * rng.uniform(-bound, bound, n)) @ Q.T
    return 0.5 * (M + M.T)


def oz_gemm(lib, A, B, use_e=0, beta=0.0, digits=False, ec=2):
    nmat, ld, _ = A.shape
    Cg = np.zeros_like(A)
    Cd = np.zeros((nmat, KS, ld, ld), dtype=np.int8) if digits else None
    ms = C.c_double(0)
    rc = lib.tp_oz_gemm(ld, nmat, A.ctypes.data_as(_dp), 1, B.ctypes.data_as(_dp), 1, use_e, 1.0, beta,
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
        assert np.array_equal(Cg[m], emulate(A[m], 1, B[m], 1))  # bit for bit
        ex = A[m] @ B[m]
        ex = np.tril(ex) + np.tril(ex, -1).T
        assert np.max(np.abs(Cg[m] - ex)) < 1e-12 * np.abs(ex).max()
        assert np.array_equal(Cg[m], Cg[m].T)                     # exactly symmetric


def test_oz_gemm_epilogue_e_term(lib):
    rng = np.random.default_rng(7)
    A = np.stack([sym(rng, 256, 1.2) for _ in range(2)])
    B = np.stack([sym(rng, 256, 1.4) for _ in range(2)])
    Cg, _ = oz_gemm(lib, A, B, use_e=1, beta=0.5)
    for m in range(2):
        want = emulate(A[m], 1, B[m], 1) + 0.5 * A[m]
        assert np.max(np.abs(Cg[m] - want)) <= 4e-16 * np.abs(want).max()


def test_oz_digit_planes_output(lib):
    # the epilogue's digit planes reconstruct its own FP64 output to 2^-57 2^e
    rng = np.random.default_rng(11)
    A = np.stack([sym(rng, 256, 1.2) for _ in range(2)])
    Cg, Cd = oz_gemm(lib, A, A, digits=True, ec=2)
    assert np.abs(Cd.astype(np.int32)).max() <= 127
    for m in range(2):
        rec = sum(Cd[m, s].astype(np.float64) * 2.0 ** (-7 * (s + 1)) for s in range(KS)) * 4.0
        assert np.max(np.abs(rec - Cg[m])) <= 2.0 ** -57 * 4.0
        assert np.array_equal(Cd[m], np.transpose(Cd[m], (0, 2, 1)))  # symmetric planes


def test_oz_gemm_deterministic(lib):
    rng = np.random.default_rng(3)
    A = np.stack([sym(rng, 384, 1.2) for _ in range(2)])
    C1, D1 = oz_gemm(lib, A, A, digits=True)
    C2, D2 = oz_gemm(lib, A, A, digits=True)
    assert np.array_equal(C1, C2) and np.array_equal(D1, D2)


@pytest.mark.parametrize("n", [200, 384])
def test_cone_projection_ozaki_vs_dmma_and_lapack(T, O, n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n))
    M = M + M.T
    M[: n // 3, : n // 3] *= 1e-6          # a cluster of small eigenvalues
    old = os.environ.get("TPB_CONE")
    try:
        os.environ["TPB_CONE"] = "ozaki"
        p_oz = T.project_psd(M)
        os.environ["TPB_CONE"] = "dmma"
        p_dm = T.project_psd(M)
    finally:
        if old is None:
            os.environ.pop("TPB_CONE", None)
        else:
            os.environ["TPB_CONE"] = old
    ref = O.project_psd(M)
    scale = np.linalg.norm(M)
    assert np.max(np.abs(p_oz - ref)) < 1e-12 * scale
    assert np.max(np.abs(p_dm - ref)) < 1e-12 * scale
    assert np.max(np.abs(p_oz - p_oz.T)) == 0.0


def test_persistent_variant_bitwise_equal():
    """The opt-in persistent kernel (TPB_OZ_PERSIST=2: 128 x 32 tiles,
    double-buffered TMEM) must reproduce the default kernel bit for bit; the
    switch is read once per process, so each variant runs in a subprocess."""
    import subprocess
    import sys

    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, ctypes as C; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "from paper_2512_07536_b200 import _lib; from test_gpu_ozaki import oz_gemm, sym;"
        "lib = _lib.load(); out = [];"
        "[out.extend(oz_gemm(lib, np.stack([sym(np.random.default_rng(ld), ld, 1.2)] * 2),"
        " np.stack([sym(np.random.default_rng(ld + 1), ld, 1.4)] * 2), digits=True)) for ld in (256, 1024)];"
        "np.save(sys.argv[1], np.concatenate([o.astype(np.float64).ravel() for o in out]))"
    )
    res = {}
    for mode in ("0", "2"):
        path = os.path.join(here, f"gpurun_out_persist_{mode}.npy")
        env = dict(os.environ, TPB_OZ_PERSIST=mode)
        subprocess.run([sys.executable, "-c", code, path], cwd=here, env=env, check=True, timeout=300)
        res[mode] = np.load(path)
        os.remove(path)
    assert res["0"].shape == res["2"].shape
    assert np.array_equal(res["0"], res["2"])
