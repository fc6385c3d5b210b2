"""CPU proofs of the bit tricks the CUDA lookup kernel relies on.

* the A/B-table PRMT encoding (csrc/gemv.cu header comment): for every
  int8 table value Q in [-127, 127], mirror flag s and slot eff,
  A + B == sigma*Q - 1 -- checked exhaustively with a bit-level model of
  `prmt.b32` (default mode: selector bit 3 replicates the selected byte's
  sign);
* the A/Y form the kernels use: prmt(~a, sel) == ~prmt(a, sel), so
  A - prmt(a, x ^ 8) == sigma*Q exactly (the B table is never stored);
* the dp2a packing: A bytes with unsigned multipliers (1, 32768), Y bytes
  with signed (-1, -32768) -> two exact stream sums in one int32, recovered
  for any group of up to 128 k-groups;
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


def test_ay_form_exhaustive():
    """prmt of the complemented table == complement of prmt, for every byte
    and selector nibble (sign-replicate mode included); hence A - Y = sQ."""
    for v in range(256):
        for nib in range(16):
            words = [(v << (8 * (nib & 3))) & 0xFFFFFFFF] * 2
            sel = nib
            lhs = prmt((~words[0]) & 0xFFFFFFFF, (~words[1]) & 0xFFFFFFFF, sel) & 0xFF
            rhs = (~prmt(words[0], words[1], sel)) & 0xFF
            assert lhs == rhs, (v, nib)
    for Q in range(-127, 128):
        a = encode_a(Q)
        for eff in range(8):
            tab_a = [(eff * 37 + j * 11) & 0xFF for j in range(8)]
            tab_a[eff] = a
            ta0 = sum(tab_a[i] << (8 * i) for i in range(4))
            ta1 = sum(tab_a[4 + i] << (8 * i) for i in range(4))
            for s in (0, 1):
                x = (s << 3) | eff
                A = s8(prmt(ta0, ta1, x) & 0xFF)
                Y = s8(prmt(ta0, ta1, x ^ 0x8) & 0xFF)
                assert A - Y == (-Q if s else Q), (Q, eff, s)


def test_mirror_encoding_matches_reference_flip():
    # x = idx ^ (7 * (idx >> 3)) gives (s, eff) with eff = idx ^ (15*s)
    # restricted to 3 bits (_kernels.py:175-176); the encoding is an involution
    for idx in range(16):
        x = idx ^ (7 * (idx >> 3))
        s, eff = x >> 3, x & 7
        assert s == idx >> 3
        assert eff == (idx ^ (15 * (idx >> 3)))
        assert (x ^ (7 * (x >> 3))) == idx


def dp2a(mult_lo: int, mult_hi: int, b: int, c: int, half: int) -> int:
    """dp2a.lo (half = 0) / .hi (half = 1) with integer multipliers and signed bytes of b."""
    b0 = s8((b >> (16 * half)) & 0xFF)
    b1 = s8((b >> (16 * half + 8)) & 0xFF)
    return int(np.int32(c + mult_lo * b0 + mult_hi * b1))


@pytest.mark.parametrize("gpg", [4, 8, 16, 32, 64, 128])
def test_dp2a_pair_packing(gpg):
    """A bytes with unsigned (1, 32768), Y bytes with signed (-1, -32768):
    acc = X + 32768 Y' with X, Y' the exact sums of sQ of two streams."""
    rng = np.random.default_rng(gpg)
    for it in range(300):
        acc, xe, xo = 0, 0, 0
        for _ in range(gpg):
            # one byte pair per stream: A and Y with A - Y = sQ in [-127, 127]
            A = rng.integers(-128, 128, 2)
            sq = rng.integers(-127, 128, 2) if it % 3 else np.array([-127, 127])
            Y = A - sq
            ok = (Y >= -128) & (Y <= 127)
            A = np.where(ok, A, sq)
            Y = np.where(ok, Y, 0)
            wa = (int(A[0]) & 0xFF) | ((int(A[1]) & 0xFF) << 8)
            wy = (int(Y[0]) & 0xFF) | ((int(Y[1]) & 0xFF) << 8)
            acc = dp2a(1, 32768, wa, acc, 0)
            acc = dp2a(-1, -32768, wy, acc, 0)
            xe += int(A[0] - Y[0])
            xo += int(A[1] - Y[1])
        v = acc
        pe = ((v << 17) & 0xFFFFFFFF)
        pe = pe - (1 << 32) if pe & 0x80000000 else pe
        pe >>= 17
        po = (v - pe) >> 15
        assert pe == xe and po == xo, (pe, xe, po, xo)


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


# ---- layer-set layout (csrc/layout.cuh, b1_core.cuh reduce_lanes_perm) ----

def perm_mask(lane: int, nidx: int) -> int:
    """b1_core.cuh perm_mask<NIDX> / layout.cuh layer_set_cmask."""
    m, o, n = 0, 1, nidx >> 1
    while n >= 1:
        if lane & o:
            m |= n
        o, n = o << 1, n >> 1
    return m


def shr16_idp(x: int) -> int:
    """common.cuh shr16_idp: dp2a.hi.u32.u32 with 16-bit multipliers (1, 256)."""
    return ((x >> 16) & 0xFF) * 1 + ((x >> 24) & 0xFF) * 256


def test_shr16_idp_is_a_shift():
    rng = np.random.default_rng(0)
    for x in rng.integers(0, 1 << 32, 2000, dtype=np.uint64):
        assert shr16_idp(int(x)) == int(x) >> 16


@pytest.mark.parametrize("nacc,lg", [(16, 1), (16, 2), (16, 4), (16, 8), (16, 16), (8, 1), (8, 4), (8, 16), (32, 4)])
def test_select_free_halving_reduces_every_index(nacc, lg):
    """A warp of 32 lanes, lane l holding logical index i ^ perm_mask(l) at
    value index i (what the lane-permuted chunks give the lookup core): the
    select-free halving (keep the low half, send the high half, first over
    the lg lanes of a quantization group, then over the groups) leaves lane l
    with the complete sum of logical index perm_mask(l), and every partial
    sum only ever adds values of ONE logical index."""
    rng = np.random.default_rng(nacc * 100 + lg)
    vals = rng.integers(-1000, 1000, (32, nacc))            # [lane][logical index]
    # v[lane][i] = (logical index, group set, sum)
    v = [[(i ^ perm_mask(l, nacc), vals[l][i ^ perm_mask(l, nacc)]) for i in range(nacc)] for l in range(32)]
    n, o = nacc, 1
    while o < 32:
        if n > 1:
            n >>= 1
            nv = [[None] * nacc for _ in range(32)]
            for l in range(32):
                for i in range(n):
                    a, b = v[l][i], v[l ^ o][i + n]
                    assert a[0] == b[0], "partner sends a different logical index"
                    nv[l][i] = (a[0], a[1] + b[1])
            v = nv
        else:
            v = [[(v[l][0][0], v[l][0][1] + v[l ^ o][0][1])] + [None] * (nacc - 1) for l in range(32)]
        o <<= 1
    # lanes that differ only in bits above log2(nacc) all hold the same index: the total is over 32 lanes
    for l in range(32):
        idx, s = v[l][0]
        assert idx == perm_mask(l, nacc) % nacc
        assert s == vals[:, idx].sum()
