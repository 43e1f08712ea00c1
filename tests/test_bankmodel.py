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
    """k_tile's u64 column tiles (the fallback of config 5's passes since r2): the model now
    serves 8-byte accesses half-warp by half-warp, as the hardware does, and reproduces what
    ncu measured on B200 -- 4 wavefronts per warp access (2-way inside each half-warp: the
    4 / 8 threads of two neighbouring networks share bank pairs), not the 2 a whole-warp
    model promised in r1; the linear tile_stride is no better"""
    NP, XS = bk.cols_u64_nbase(K, TQ)
    assert bk.cols_u64_worst(K, TQ, NP, XS) == 4
    assert bk.cols_u64_worst(K, TQ, tile_stride(K, TQ, 8), 0) >= 4


@pytest.mark.parametrize("K,TQ", [(5, 128), (6, 64), (7, 32), (8, 16)])
def test_u64_tensor_box_column_tiles_are_conflict_free(K, TQ):
    """colpass.cuh k_cols: dense [row][column] tiles, a warp's lanes along the columns -- every
    register-group access is 2 wavefronts (one per half-warp) under the half-warp rule, for the
    bit-reversed first gather too"""
    TT = 1 << (K - 4)
    for tid0 in range(0, 256, 32):
        for c in range(16):
            for B in (0, K - 4):
                lanes = []
                for tid in range(tid0, tid0 + 32):
                    t, u = tid % TQ, tid // TQ
                    pbase = (u & ((1 << B) - 1)) | ((u >> B) << (B + 4))
                    lanes.append((pbase | (c << B)) * TQ + t)
                assert bk.wavefronts(lanes, 8) == 2
            lanes = [(bk.brev(tid // TQ, K - 4) + (bk.brev(c, 4) << (K - 4))) * TQ + tid % TQ
                     for tid in range(tid0, tid0 + 32)]
            assert bk.wavefronts(lanes, 8) == 2
