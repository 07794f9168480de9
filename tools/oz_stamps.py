"""Phase breakdown of one Ozaki GEMM launch from globaltimer stamps
(instrumentation build: make -C paper_2512_07536_b200 STAMPS=1; GPU box):
  TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/oz_stamps.py [ld]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib  # noqa: E402

ld = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lib = _lib.load()
tiles = 2 * (ld // 128) * (ld // 128 + 1) // 2
buf = torch.zeros(8 * tiles * 2, dtype=torch.int64, device="cuda")
assert lib.tp_oz_set_stamps(C.c_void_p(buf.data_ptr())) == 0
rng = np.random.default_rng(1)
Q, _ = np.linalg.qr(rng.standard_normal((ld, ld)))
A = (Q * rng.uniform(-1.2, 1.2, ld)) @ Q.T
A = np.ascontiguousarray(np.stack([0.5 * (A + A.T)] * 2))
Cg = np.zeros_like(A)
Cd = np.zeros((2, 7, ld, ld), np.int8)
dp = C.POINTER(C.c_double)
ms = C.c_double(0)
for it in range(3):
    # reps=2: the timed repetitions write digit planes only (the cone
    # iteration's intermediate products); the stamps are the last one's
    rc = lib.tp_oz_gemm(ld, 2, A.ctypes.data_as(dp), 2, A.ctypes.data_as(dp), 2, 0, 1.0, 0.0,
                        Cg.ctypes.data_as(dp), Cd.ctypes.data_as(C.c_void_p), 3, 2, C.byref(ms))
    assert rc == 0
    torch.cuda.synchronize()
    st = buf.view(-1, 8).cpu().numpy()[:, :7].astype(np.float64)
    t0 = st[:, 0].min()
    rel = (st - t0) / 1e3  # us
    print(f"ld={ld} run {it}: CTAs {len(st)}  start spread {rel[:, 0].max():.2f} us")
    for name, a, b in (("main loop (start -> last MMA commit)", 0, 1), ("commit -> epilogue sees TMEM", 1, 2),
                       ("TMEM drain + FP64", 2, 3), ("staging + symmetrise (smem)", 3, 5), ("digit split + mirror stores", 5, 6),
                       ("direct-row stores", 6, 4), ("start -> end", 0, 4)):
        d = rel[:, b] - rel[:, a]
        print(f"  {name:40s} mean {d.mean():7.2f}  min {d.min():7.2f}  max {d.max():7.2f} us")
    print(f"  last CTA end {rel[:, 4].max():.2f} us")
