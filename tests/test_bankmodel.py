"""Shared-memory bank model of the tile kernel (tools/bankcheck.py) -- the
B200 counterpart of the reference's bankmodel tests:
replays every warp access of one tile for the shipped shapes and pins that the
exchange layout (padpos + network stride tile_stride) is conflict-free where
the design claims it is."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import bankcheck as bk  # noqa: E402


def tile_stride(K, TQ, word):
    """csrc/fasttile.cuh tile_stride<T,K,TQ>()"""
    nb = 32 if word == 4 else 16
    want = 1 if TQ >= nb else nb // TQ
    n = bk.padded_len(K, word)
    while n % nb != want:
        n += 1
    return n


def test_padpos_is_additive_over_disjoint_bits():
    for a in range(0, 1 << 10, 37):
        for b in (1 << 10, 3 << 11, 5 << 12):
            assert bk.padpos(a | b) == bk.padpos(a) + bk.padpos(b)


@pytest.mark.parametrize("V", ["dit", "pease"])
def test_u32_k10_tile_is_conflict_free(V):
    # config 4: two passes of K = 10, TQ = 8 (the shipped 2^20 plan)
    NP = tile_stride(10, 8, 4)
    for key, ratio in bk.breakdown(V, 10, 8, NP).items():
        assert ratio == 1.0, (V, key, ratio)


def test_u64_k8_tile_is_conflict_free():
    # config 3: Goldilocks 2^16 = two passes of K = 8, TQ = 16
    NP = tile_stride(8, 16, 8)
    for V in ("dif", "dit"):
        t, ideal = bk.score(V, 8, 16, bk.tile_nt(8, 16), NP, 8,
                            [(a, b, c, d, e) for (a, b, c, d, e) in bk.SHAPES[V]])
        assert t == ideal, (V, t, ideal)


def test_small_networks_conflict_as_documented():
    # K = 8 tiles (TQ = 32): 8-thread networks share warps, 2-way group conflicts
    # for any stride -- the reason 3-pass plans lose
    best = min(bk.score("dit", 8, 32, 512, NP, 4, bk.SHAPES["dit"])[0] for NP in range(264, 297))
    _, ideal = bk.score("dit", 8, 32, 512, 265, 4, bk.SHAPES["dit"])
    assert best / ideal > 1.5


@pytest.mark.parametrize("V", ["dit", "pease"])
@pytest.mark.parametrize("K", [7, 8, 9, 10])
def test_tma_fourstep_column_pass_is_conflict_free(V, K):
    """fourstep_tma.cuh TmaGeo<V, K>: the tile-major groups (dense TMA staging
    reads, padded work-buffer writes, last-group reads) of the shipped geometry"""
    import bank_fs
    assert bank_fs.worst_conflict(V, K) == 1


@pytest.mark.parametrize("K,TQ", [(7, 32), (6, 64)])
def test_u64_column_tiles_nonlinear_base(K, TQ):
    """config 5's column/row passes: the shipped base(t) = t*NP + (t >> XS) is
    conflict-free (2 wavefronts = one 256-byte warp access) where the linear
    tile_stride was 2-way conflicted"""
    NP, XS = bk.cols_u64_nbase(K, TQ)
    assert bk.cols_u64_worst(K, TQ, NP, XS) == 2
    assert bk.cols_u64_worst(K, TQ, tile_stride(K, TQ, 8), 0) > 2
