"""Shared-memory bank model of the kernels' exchange patterns (CPU only).

Re-derives, per 128-byte phase, for every compiled kernel variant (queried from the library with
sfft_variant_info), the addresses each warp instruction touches in shared
memory -- the Stockham scatter/gather of csrc/sfft_kernels.cuh with its XOR
row swizzle or padding, and the tile kernel's 16-byte chunk staging -- and counts
bank-conflict wavefronts with the 32 x 4-byte bank model.  The default
variant of every (precision, N) must be conflict-free; ncu's
l1tex__data_bank_conflicts_pipe_lsu_mem_shared counters confirm it on the GPU.
"""

import pytest

from paper_2203_09384_b200 import _native

ALL_N = [2**p for p in range(1, 12)]


def swz_row(e: int, r: int, esize: int) -> int:
    """LAYOUT 2: e ^ ((e / R) & (W - 1)), W = complex elements per 128-byte row."""
    w = 128 // esize
    return e ^ ((e // r) & (w - 1))


def swz_chunk(c: int) -> int:
    return c ^ (((c >> 3) ^ (c >> 6)) & 7)


def wavefronts(unit_idx, unit_bytes):
    """(actual, ideal) wavefronts of one warp access; unit_idx[lane] in units.

    Shared memory serves a warp in phases of 128 bytes' worth of lanes (32
    lanes for 4-byte, 16 for 8-byte, 8 for 16-byte accesses); within a phase
    every distinct 4-byte word mapped to the same bank costs one wavefront.
    """
    per = 128 // unit_bytes
    tot = 0
    for p0 in range(0, 32, per):
        words = set()
        for u in unit_idx[p0 : p0 + per]:
            for w in range(unit_bytes // 4):
                words.add(u * (unit_bytes // 4) + w)
        banks = {}
        for w in words:
            banks.setdefault(w % 32, set()).add(w)
        tot += max(len(v) for v in banks.values())
    return tot, 32 // per


def stockham_instructions(info, esize):
    """Every smem access of sfft::stockham_kernel (remainder radix last)."""
    n, r, radices, layout = info["n"], info["elems_per_thread"], info["radices"], info["layout"]
    g = n // r
    region = n + n // r  # LAYOUT 1: padded per-sequence region

    def addr(s, e):
        if layout == 1:
            return s * region + e + e // r
        if layout == 3:  # split exchange: 8-byte words, real then imaginary parts
            return swz_row(s * n + e, r, 8)
        assert layout == 2
        return swz_row(s * n + e, r, esize)

    lanes = [(lane // g, lane % g) if g < 32 else (0, lane) for lane in range(32)]
    # loader 3: the exchange feeding the last pass is scattered linearly and
    # gathered through tensor memory (tcgen05.cp), not with LDS
    tmem_last = info["loader"] == 3
    last = len(radices) - 1
    out = []
    stride = 1
    for pi, rad in enumerate(radices):
        nb = r // rad
        if pi > 0 and not (tmem_last and pi == last):  # gather x[j + m*G]
            for mm in range(r):
                out.append([addr(s, j + mm * g) for s, j in lanes])
        if pi < last:  # scatter to the Stockham destination
            linear = tmem_last and pi == last - 1
            for t in range(nb):
                for q in range(rad):
                    idx = []
                    for s, j in lanes:
                        b = j + t * g
                        k = b % stride
                        e = (b - k) * rad + k + q * stride
                        idx.append(s * n + e if linear else addr(s, e))
                    out.append(idx)
        stride *= rad
    if layout == 3:
        out = out + out  # the same pattern for the imaginary parts
    return out


def tile_instructions(n, spt, esize):
    k = n * esize // 16
    if k == 1:
        return []  # no staging
    out = []
    for i in range(spt * k):  # cp.async / coalesced chunk accesses
        out.append([swz_chunk(lane + 32 * i) for lane in range(32)])
    for u in range(spt):  # per-thread sequence accesses
        for c in range(k):
            out.append([swz_chunk((u * 32 + lane) * k + c) for lane in range(32)])
    return out


def split2_instructions(info, esize):
    """sfft::split2_kernel: each warp runs the one-warp Stockham passes of the
    N/2 transform in its own region (regions start at multiples of 128 bytes,
    so the per-warp pattern is the whole story), then the warps trade halves
    through linear [m][lane] slots.  The polyphase gather from the linear TMA
    staging is modelled separately (split2_gather)."""
    half = dict(info, n=info["n"] // 2, radices=info["radices"][:-1])
    out = stockham_instructions(half, esize)
    hr = info["elems_per_thread"] // 2
    for m in range(2 * hr):  # swap writes / reads
        out.append([m * 32 + lane for lane in range(32)])
    return out


def split2_gather(info):
    """v[m] = staging[2 (lane + 32 m) + w]: every other element of the row."""
    r = info["elems_per_thread"]
    return [[2 * (lane + 32 * m) + w for lane in range(32)] for w in (0, 1) for m in range(r)]


def fourstep_instructions(info):
    """sfft::fourstep_kernel (fp64 N = 2048, 128 threads): the staging gather
    v[a] = x[n1 + 32 (4 a + c0 + 2 c1)], the transpose write slot(n1, k2) =
    64 n1 + (k2 ^ (n1 & 7)) for k2 = i + 8 c1 + 16 c0 + 32 h, and its read by
    thread (k2, d) of n1 = 2 b + d.  Lane l of warp w: c0 = bit 3, c1 = bit 4,
    n1 = (l & 7) + 8 w; after the transpose k2 = (l & 15) + 16 w, d = bit 4."""
    out = []
    for w in range(4):
        quad = [((l >> 3) & 1, (l >> 4) & 1, (l & 7) + 8 * w) for l in range(32)]
        for a in range(16):
            out.append([n1 + 32 * (c0 + 2 * c1) + 128 * a for c0, c1, n1 in quad])
        for h in (0, 1):
            for i in range(8):
                out.append([64 * n1 + ((i + 8 * c1 + 16 * c0 + 32 * h) ^ (n1 & 7)) for c0, c1, n1 in quad])
        pairs = [((l & 15) + 16 * w, (l >> 4) & 1) for l in range(32)]
        for b in range(16):
            out.append([64 * (2 * b + d) + (k2 ^ ((2 * b + d) & 7)) for k2, d in pairs])
    return out


def conflict_ratio(info, esize):
    if info["kernel"] == _native.SFFT_KERNEL_FOURSTEP:
        instrs = fourstep_instructions(info)
        unit = esize
    elif info["kernel"] == _native.SFFT_KERNEL_STOCKHAM:
        instrs = stockham_instructions(info, esize)
        unit = 8 if info["layout"] == 3 else esize
    elif info["kernel"] == _native.SFFT_KERNEL_SPLIT2:
        instrs = split2_instructions(info, esize)
        unit = esize
    else:
        spt = info["seqs_per_cta"] // info["threads_per_cta"]
        instrs = tile_instructions(info["n"], spt, esize)
        unit = 16
    if not instrs:
        return 1.0
    tot = ideal = 0
    for idx in instrs:
        a, b = wavefronts(idx, unit)
        tot += a
        ideal += b
    return tot / ideal


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("n", ALL_N)
def test_default_variant_conflict_free(n, prec):
    info = _native.variant_info(n, prec, 0)
    assert conflict_ratio(info, 8 if prec == 0 else 16) == 1.0


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("n", ALL_N)
def test_every_variant_bounded(n, prec):
    lib = _native.lib()
    for v in range(lib.sfft_num_variants(n, prec)):
        info = _native.variant_info(n, prec, v)
        assert conflict_ratio(info, 8 if prec == 0 else 16) <= 2.0


def test_split2_gather_is_exactly_two_way():
    """The one documented conflict: the polyphase gather reads 16-byte elements
    at a 32-byte stride (2 wavefronts per 8-lane phase instead of 1); every
    exchange and the half swap are conflict-free (conflict_ratio == 1)."""
    lib = _native.lib()
    seen = 0
    for prec in (0, 1):
        for n in ALL_N:
            for v in range(lib.sfft_num_variants(n, prec)):
                info = _native.variant_info(n, prec, v)
                if info["kernel"] != _native.SFFT_KERNEL_SPLIT2:
                    continue
                esize = 8 if prec == 0 else 16
                assert conflict_ratio(info, esize) == 1.0
                tot = ideal = 0
                for idx in split2_gather(info):
                    a, b = wavefronts(idx, esize)
                    tot, ideal = tot + a, ideal + b
                assert tot == 2 * ideal
                seen += 1
    assert seen >= 1


def test_split_exchange_variant_conflict_free():
    """LAYOUT 3 (fp64, real then imaginary parts through 8-byte words) is
    conflict-free wherever it is compiled."""
    lib = _native.lib()
    seen = 0
    for n in ALL_N:
        for v in range(lib.sfft_num_variants(n, 1)):
            info = _native.variant_info(n, 1, v)
            if info["kernel"] == _native.SFFT_KERNEL_STOCKHAM and info["layout"] == 3:
                assert conflict_ratio(info, 16) == 1.0
                seen += 1
    assert seen >= 1


def test_tmem_gather_variant_conflict_free():
    """Loader 3 (fp64 N=2048: the last exchange scattered to a linear buffer
    and gathered through tensor memory): the linear scatter of the Stockham
    pattern writes 8 consecutive 16-byte elements per phase -- conflict-free
    without a swizzle -- and the remaining LDS/STS stay conflict-free."""
    lib = _native.lib()
    seen = 0
    for v in range(lib.sfft_num_variants(2048, 1)):
        info = _native.variant_info(2048, 1, v)
        if info["loader"] == 3:
            assert conflict_ratio(info, 16) == 1.0
            seen += 1
    assert seen >= 1


def test_swizzles_are_bijections():
    for esize, rs in ((8, (16, 32)), (16, (8, 16, 32))):
        for r in rs:
            assert sorted(swz_row(e, r, esize) for e in range(4096)) == list(range(4096))
    assert sorted(swz_chunk(c) for c in range(4096)) == list(range(4096))


def test_fourstep_variant_conflict_free():
    """The four-step kernel's gather, transpose write and transpose read are
    conflict-free (its radix-2 level moves through shuffles, not shared memory)."""
    lib = _native.lib()
    seen = 0
    for v in range(lib.sfft_num_variants(2048, 1)):
        info = _native.variant_info(2048, 1, v)
        if info["kernel"] == _native.SFFT_KERNEL_FOURSTEP:
            assert conflict_ratio(info, 16) == 1.0
            seen += 1
    assert seen >= 1
