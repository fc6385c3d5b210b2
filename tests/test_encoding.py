"""CPU proofs of the bit tricks the CUDA lookup kernel relies on.

* the A/B-table PRMT encoding (csrc/gemv.cu header comment): for every
  int8 table value Q in [-127, 127], mirror flag s and slot eff,
  A + B == sigma*Q - 1 -- checked exhaustively with a bit-level model of
  `prmt.b32` (default mode: selector bit 3 replicates the selected byte's
  sign);
* the dp2a packing: two streams in one int32 with multipliers (1, -32768)
  are recovered exactly for any group of up to 128 k-groups;
* layout v2 (csrc/layout.cuh): the chunk offset map is a bijection onto
  [0, bits*M*K/8) for every BASELINE shape.
"""
import numpy as np
import pytest


def prmt(a: int, b: int, sel: int) -> int:
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    out = 0
    for n in range(4):
        nib = (sel >> (4 * n)) & 0xF
        byte = src[nib & 7]
        if nib & 8:
            byte = 0xFF if byte & 0x80 else 0x00
        out |= byte << (8 * n)
    return out


def s8(x: int) -> int:
    return x - 256 if x & 0x80 else x


def encode_a(q: int) -> int:
    return (q - (1 if q < 0 else 0)) & 0xFF


def test_ab_trick_exhaustive():
    for Q in range(-127, 128):
        a = encode_a(Q)
        b = (~a) & 0xFF
        for eff in range(8):
            # put Q at slot eff, random junk elsewhere
            tab_a = [(eff * 37 + j * 11) & 0xFF for j in range(8)]
            tab_a[eff] = a
            tab_b = [(~v) & 0xFF for v in tab_a]
            ta0 = sum(tab_a[i] << (8 * i) for i in range(4))
            ta1 = sum(tab_a[4 + i] << (8 * i) for i in range(4))
            tb0 = sum(tab_b[i] << (8 * i) for i in range(4))
            tb1 = sum(tab_b[4 + i] << (8 * i) for i in range(4))
            for s in (0, 1):
                x = (s << 3) | eff
                A = s8(prmt(ta0, ta1, x) & 0xFF)
                B = s8(prmt(tb0, tb1, x ^ 0x8) & 0xFF)
                sigma = -1 if s else 1
                assert A + B == sigma * Q - 1, (Q, eff, s, A, B)


def test_mirror_encoding_matches_reference_flip():
    # x = idx ^ (7 * (idx >> 3)) gives (s, eff) with eff = idx ^ (15*s)
    # restricted to 3 bits (_kernels.py:175-176); the encoding is an involution
    for idx in range(16):
        x = idx ^ (7 * (idx >> 3))
        s, eff = x >> 3, x & 7
        assert s == idx >> 3
        assert eff == (idx ^ (15 * (idx >> 3)))
        assert (x ^ (7 * (x >> 3))) == idx


@pytest.mark.parametrize("gpg", [4, 8, 16, 32, 64, 128])
def test_dp2a_pair_packing(gpg):
    rng = np.random.default_rng(gpg)
    M = -32768
    for _ in range(2000):
        # per-lookup contributions A+B in [-128, 126]
        xe = rng.integers(-128, 127, gpg)
        xo = rng.integers(-128, 127, gpg)
        if _ % 3 == 0:
            xe[:] = -128
            xo[:] = 126
        acc = int(np.int32(np.sum(xe) + M * np.sum(xo)))
        v = acc + (-32767 * gpg)          # add back +1 per lookup on both streams
        v = int(np.int32(v))
        pe = ((v << 17) & 0xFFFFFFFF)
        pe = pe - (1 << 32) if pe & 0x80000000 else pe
        pe >>= 17
        po = (pe - v) >> 15
        assert pe == int(np.sum(xe)) + gpg and po == int(np.sum(xo)) + gpg


def chunk_offsets(m, k, bits, gs):
    tile_ch = 32 if bits == 3 else 32 // bits
    n_sg = 3 if bits == 3 else 1
    gpg = gs // 4
    R = 8 if gpg % 8 == 0 else 4
    KG = k // 4
    U = KG // R
    n_tiles = m // tile_ch
    kg = np.arange(KG)
    u, r = kg // R, kg % R
    ub, l = u >> 5, u & 31
    nu_b = np.minimum(32, U - 32 * ub)
    within = ub * (32 * R * 16) + (r * nu_b + l) * 16
    rows = np.arange(n_tiles * n_sg)[:, None] * KG * 16
    return (rows + within[None, :]).reshape(-1)


@pytest.mark.parametrize("m,k,bits,gs", [
    (4096, 4096, 2, 64), (11008, 4096, 2, 64), (4096, 11008, 2, 64), (4096, 4096, 4, 128),
    (4096, 4096, 1, 128), (8192, 28672, 2, 128), (1024, 8192, 4, 128), (96, 512, 3, 64),
    (64, 256, 4, 32), (32, 1024, 1, 16),
])
def test_layout_v2_bijection(m, k, bits, gs):
    off = chunk_offsets(m, k, bits, gs)
    total = m * bits * k // 8
    assert off.size * 16 == total
    assert off.min() == 0 and off.max() == total - 16
    assert np.all(off % 16 == 0)
    assert np.unique(off).size == off.size
