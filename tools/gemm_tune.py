"""Time the DMMA GEMM variants (tp_bench_gemm) at the workload shapes."""
import ctypes as C
import sys
sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib
L = _lib.load()
for n, nmat in [(1024, 2), (256, 512), (512, 2), (2048, 2)]:
    ld = (n + 63) // 64 * 64
    tiles = (ld // 64) * (ld // 64 + 1) // 2
    flops = nmat * tiles * 64 * 64 * ld * 2.0
    for v in range(5 if nmat == 2 else 4):
        ms = C.c_double()
        rc = L.tp_bench_gemm(n, nmat, v, 20, C.byref(ms))
        print(f"n={n:5d} nmat={nmat:4d} variant={v} rc={rc} {ms.value*1e3:9.1f} us  {flops/ms.value/1e9:6.2f} TFLOP/s (tile flops)")
