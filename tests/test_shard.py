"""CPU: host logic of the sharded single-instance projection (SURVEY §8e,
ozaki_kernels.cuh OzShard). The ranks' tile lists partition the lower tiles
(round-robin, balanced), and since every rank's epilogue stores its tiles
into every rank's buffer, the union of their footprints under the kernel's
store rule (lower tiles (I, J), J < 2(I+1), of 128 x 64; direct rows from
64 t in the diagonal block, mirror rows from 64 (t+1)) writes every entry of
the iterate exactly once; the GPU check (bitwise equality with the
single-GPU solve at 2 ranks) is tests/test_gpu_shard.py.""",
import numpy as np
import pytest

BM, BN, R = 128, 64, 2


def tile_of(t):
    I = 0
    while R * (I + 1) * (I + 2) // 2 <= t:
        I += 1
    return I, t - R * I * (I + 1) // 2


def footprint(ld, tiles):
    """Entries of the ld x ld iterate the listed tiles write (kernel store rule)."""
    W = np.zeros((ld, ld), np.int32)
    for t in tiles:
        I, J = tile_of(int(t))
        i0, j0 = I * BM, J * BN
        td = J - R * I
        dr0 = 0 if td < 0 else BN * td
        mr0 = 0 if td < 0 else BN * (td + 1)
        W[i0 + dr0:i0 + BM, j0:j0 + BN] += 1                 # direct rows
        W[j0:j0 + BN, i0 + mr0:i0 + BM] += 1                 # mirror (transposed)
    return W


@pytest.mark.parametrize("ld,G", [(256, 2), (512, 2), (512, 4), (1024, 2), (1024, 8), (2048, 4), (384, 2)])
def test_shard_tiles_partition_the_iterate(T, ld, G):
    all_lower = R * (ld // BM) * (ld // BM + 1) // 2
    single = footprint(ld, range(all_lower))
    assert (single == 1).all()                               # unsharded: every entry once
    union = np.zeros_like(single)
    seen = set()
    sizes = []
    for k in range(G):
        t = T.shard_tiles(ld, G, k)
        assert len(t) == len(set(t.tolist())) and t.min() >= 0 and t.max() < all_lower
        assert not (seen & set(t.tolist()))                  # disjoint
        seen |= set(t.tolist())
        sizes.append(len(t))
        union += footprint(ld, t)
    assert len(seen) == all_lower                            # every tile on some rank
    assert max(sizes) - min(sizes) <= 1                      # balanced
    assert (union == 1).all()                                # every entry written once


def test_shard_tiles_rejects_bad_ranks(T):
    with pytest.raises(Exception):
        T.shard_tiles(512, 9, 0)                             # more than 8 ranks
    with pytest.raises(Exception):
        T.shard_tiles(500, 2, 0)                             # ld not a multiple of 128
