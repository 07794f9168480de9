"""Ozaki-scheme tcgen05 GEMM (tp_oz_gemm) vs an exact numpy emulation and
vs FP64 numpy; timing per launch. Run on a GPU box:
    python tools/oz_check.py [ld ...]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib  # noqa: E402

sys.path.insert(0, "tests")
from test_gpu_ozaki import KS, emulate  # noqa: E402  (balanced base-256 digit emulation)


def sym_matrix(rng, n, bound):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = rng.uniform(-bound, bound, n)
    M = (Q * ev) @ Q.T
    return 0.5 * (M + M.T)


def run(ld, nmat=2, reps=20, use_e=0, beta=0.0):
    lib = _lib.load()
    rng = np.random.default_rng(ld)
    A = np.stack([sym_matrix(rng, ld, 1.2) for _ in range(nmat)])
    B = np.stack([sym_matrix(rng, ld, 1.4) for _ in range(nmat)])
    Cg = np.zeros_like(A)
    Cd = np.zeros((nmat, KS, ld, ld), dtype=np.int8)
    ms = C.c_double(0)
    dp = C.POINTER(C.c_double)
    rc = lib.tp_oz_gemm(ld, nmat, A.ctypes.data_as(dp), 2, B.ctypes.data_as(dp), 2, use_e, 1.0, beta,
                        Cg.ctypes.data_as(dp), Cd.ctypes.data_as(C.c_void_p), 3, reps, C.byref(ms))
    if rc != 0:
        raise RuntimeError(lib.tp_last_error_message().decode() if hasattr(lib, "tp_last_error_message") else rc)
    worst_emu = worst_fp = worst_dig = 0.0
    for m in range(nmat if not os.environ.get("OZ_NOEMU") else 0):
        emu = emulate(A[m], 2, B[m], 2) + (beta * A[m] if use_e else 0.0)
        ex = A[m] @ B[m]
        ex = np.tril(ex) + np.tril(ex, -1).T + (beta * A[m] if use_e else 0.0)
        sc = np.abs(ex).max()
        worst_emu = max(worst_emu, np.abs(Cg[m] - emu).max() / sc)
        worst_fp = max(worst_fp, np.abs(Cg[m] - ex).max() / sc)
        rec = sum(Cd[m, s].astype(np.float64) * 2.0 ** (-8 * (s + 1)) for s in range(KS)) * 8.0
        worst_dig = max(worst_dig, np.abs(rec - Cg[m]).max())
    tiles = 2 * (ld // 128) * (ld // 128 + 1) // 2  # 128 x 64 lower tiles
    ops = 2.0 * 128 * 64 * ld * (KS * (KS + 1) // 2) * tiles * nmat  # int8 MACs x 2
    print(f"ld={ld:5d} nmat={nmat} |C-emu|/max={worst_emu:.2e} |C-fp64|/max={worst_fp:.2e} "
          f"|digits-C|={worst_dig:.2e}  {ms.value * 1e3:8.1f} us/launch  "
          f"int8 {ops / ms.value / 1e9:7.1f} TOP/s  fp64-equiv {2.0 * ld ** 3 * nmat / 2 / ms.value / 1e9:6.1f} TFLOP/s",
          flush=True)
    return worst_emu, worst_fp


if __name__ == "__main__":
    # arguments: ld or ld:nmat (OZ_NOEMU=1 skips the emulation checks: timing only)
    lds = sys.argv[1:] or ["128", "256", "512", "1024"]
    for a in lds:
        ld, _, nm = a.partition(":")
        run(int(ld), nmat=int(nm) if nm else 2)
    run(256, use_e=1, beta=0.5)
