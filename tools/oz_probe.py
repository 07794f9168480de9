"""Phase breakdown of the Ozaki GEMM (globaltimer stamps per CTA) under the
instrumentation modes: 0 full, 1 no MMA, 2 no TMA, 3 neither."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib  # noqa: E402
from tools.oz_check import sym_matrix  # noqa: E402

lib = _lib.load()
DIG = '--digits' in sys.argv
sys.argv = [a for a in sys.argv if a != '--digits']
dp = C.POINTER(C.c_double)
args = [int(a) for a in sys.argv[1:]]
modes = (args[1],) if len(args) > 1 else (0, 1, 2, 3)
for ld in args[:1] or [128, 1024]:
    rng = np.random.default_rng(1)
    nmat = 2
    A = np.stack([sym_matrix(rng, ld, 1.2) for _ in range(nmat)])
    Cg = np.zeros_like(A)
    Cd = np.zeros((nmat, 8, ld, ld), dtype=np.int8)
    tiles = 2 * (ld // 128) * (ld // 128 + 1) // 2
    for mode in modes:
        st = np.zeros((nmat * tiles, 8), dtype=np.int64)
        ms = C.c_double(0)
        rc = lib.tp_oz_gemm_dbg(ld, nmat, A.ctypes.data_as(dp), 1, A.ctypes.data_as(dp), 1, 0, 1.0, 0.0,
                                Cg.ctypes.data_as(dp), Cd.ctypes.data_as(C.c_void_p) if DIG else None, 2, 10, C.byref(ms), mode,
                                st.ctypes.data_as(C.c_void_p))
        assert rc == 0, lib.tp_last_error_message()
        t0 = st[:, 0].min()
        setup = np.median(st[:, 1] - st[:, 0]) / 1e3
        main = np.median(st[:, 2] - st[:, 1]) / 1e3
        epi = np.median(st[:, 3] - st[:, 2]) / 1e3
        span = (st[:, 3].max() - t0) / 1e3
        launch_skew = (st[:, 0].max() - t0) / 1e3
        acc = np.median(st[:, 4] - st[:, 2]) / 1e3
        stg = np.median(st[:, 5] - st[:, 4]) / 1e3
        cst = np.median(st[:, 6] - st[:, 5]) / 1e3
        dig = np.median(st[:, 3] - st[:, 6]) / 1e3
        print(f"   epi: tmem->acc {acc:5.2f} stage {stg:5.2f} C-stores {cst:5.2f} digits {dig:5.2f} us")
        print(f"ld={ld:5d} mode={mode} {ms.value*1e3:7.1f} us/launch | CTA: setup {setup:6.2f} main {main:7.2f} "
              f"epi {epi:6.2f} us | span {span:7.2f} start-skew {launch_skew:6.2f}", flush=True)
