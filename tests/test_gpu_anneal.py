"""GPU: the device warm-start annealer (anneal_kernels.cu) reproduces the
reference's random stream and decisions: its mt19937_64 against a pure-Python
std::mt19937_64, and its edge sets against the host port of the same loop
(and, via test_gpu_solve, against the reference's own warm starts)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def mt19937_64(seed, k):
    """std::mt19937_64 (the standard's parameters), first k outputs."""
    x = [seed & M64]
    for i in range(1, 312):
        x.append((6364136223846793005 * (x[-1] ^ (x[-1] >> 62)) + i) & M64)
    out, idx = [], 312
    for _ in range(k):
        if idx >= 312:
            for i in range(312):
                y = (x[i] & 0xFFFFFFFF80000000) | (x[(i + 1) % 312] & 0x7FFFFFFF)
                x[i] = x[(i + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            idx = 0
        y = x[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & M64
        y ^= (y << 37) & 0xFFF7EEE000000000 & M64
        y ^= y >> 43
        out.append(y & M64)
    return out


def test_device_mt19937_64():
    from paper_2512_07536_b200 import _lib
    lib = _lib.load()
    for seed in (0, 5489, 2 ** 63 + 17):
        out = (C.c_uint64 * 700)()
        assert lib.tp_device_mt19937_64(seed, 700, out) == 0
        assert list(out) == mt19937_64(seed, 700)


@pytest.mark.parametrize("n,deg,steps,seed", [(16, 4, 20, 0), (64, 6, 8, 3), (100, 5, 3, 7), (300, 8, 1, 1)])
def test_device_anneal_equals_reference(T, n, deg, steps, seed):
    """Device annealer vs the compiled reference's anneal_degree_topology
    (oracle/_ref): identical edge sets."""
    from oracle import ref
    degrees = [deg] * n
    if (deg * n) % 2:
        degrees[0] += 1
    dev = T.anneal_degree_topology(degrees, steps=steps, seed=seed)
    want = ref.anneal_degree(degrees, steps=steps, seed=seed)
    assert np.array_equal(np.asarray(dev).reshape(-1, 2), np.asarray(want).reshape(-1, 2))


def test_device_anneal_heterogeneous(T, O):
    from oracle import ref
    bu, e = O.allocate_edge_capacity([9.76] * 16 + [3.25] * 16, 64)
    dev = T.anneal_degree_topology(e, steps=10, seed=2)
    want = ref.anneal_degree(e, steps=10, seed=2)
    assert np.array_equal(np.asarray(dev).reshape(-1, 2), np.asarray(want).reshape(-1, 2))
