"""Model check of the 16x16 raster's fixed-point arithmetic (csrc/hht_kernels.cu, Raster16; DESIGN.md
§4): the kernel's integer formulas, restated here, reproduce floor(y_u / 3N) exactly at every
column of every line that crosses a level-(D-4) region, and its table (indexed by the sum of two
consecutive floors) selects exactly the cells the paper's corner test marks as crossed
(G_SW > 0 >= G_NE). Pure integer host arithmetic; no GPU, no oracle."""
import random

import pytest


def fx_consts(N):
    """The host constants of pass_args (csrc/hht_driver.cu)."""
    n3 = 3 * N
    s = 0
    while (1 << s) < 32 * n3:
        s += 1
    return s, ((1 << (24 + s)) + n3 - 1) // n3, (1 << (24 + s)) // n3


def rows_of_entry(t):
    """Rows of table entry t = f_u + f_(u+1) (tab16_entry)."""
    f = (t + 1) // 2 if t >= 0 else -((-t) // 2)
    fn = t - f
    return set(range(max(fn, 0), min(f, 15) + 1))


@pytest.mark.parametrize("N", [1, 2, 3, 16, 64, 511, 512, 1000, 4096, 8192, 32767])
def test_fixed_point_floor_exact(N):
    s, m, mlo = fx_consts(N)
    assert m < (1 << 32) and (1 << 24) // (3 * N) > 34
    n3 = 3 * N
    r = random.Random(N)
    for trial in range(4000):
        ex = r.randrange(N)
        lim = 16 * (2 * ex + n3)                  # G_SW - 1 of a line crossing the 16x16 region
        y0 = r.randrange(lim) if trial % 3 else (r.randrange(27) * n3) % lim
        B = r.randrange(17, 146)                  # the per-block bias (tab16_place)
        Y = ((y0 * m) >> s) + 1 + (B << 24)
        P = (2 * ex * mlo) >> s
        for u in range(17):
            Yu = (Y - u * P) & 0xFFFFFFFF
            assert (Yu >> 24) - B == (y0 - u * 2 * ex) // n3, (N, ex, y0, u)


@pytest.mark.parametrize("N", [4, 16, 512, 8192])
def test_table_rows_match_corner_test(N):
    n3 = 3 * N
    r = random.Random(7 + N)
    for _ in range(1500):
        ex = r.randrange(N)
        y0 = r.randrange(16 * (2 * ex + n3))
        for u in range(16):
            yu, yn = y0 - 2 * ex * u, y0 - 2 * ex * (u + 1)
            direct = {v for v in range(16) if yu - n3 * v >= 0 and yn - n3 * (v + 1) < 0}
            assert rows_of_entry(yu // n3 + yn // n3) == direct
    assert rows_of_entry(-2) == set()             # lanes past the batch: f = -1 in every column


@pytest.mark.parametrize("N,D", [(1, 5), (3, 5), (64, 6), (512, 9), (8192, 13), (32767, 15), (65536, 20)])
def test_setup_multiply_high(N, D):
    """Raster16::run's setup: y0 2^k (k = 32 - fx_s) formed in 32-bit modular arithmetic from the
    per-batch constants (alpha 2^k, 2^(D+k) mod 2^32, (beta - 1) 2^k), then Y_0 = mulhi(y0 2^k, fx_m)
    + bias and P = mulhi(ex 2^(k+1), fx_mlo) equal the 64-bit forms floor(y0 fx_m / 2^fx_s) and
    floor(2ex fx_mlo / 2^fx_s) for every line crossing a level-(D-4) region (0 <= y0 < 2^fx_s)."""
    s, m, mlo = fx_consts(N)
    k = 32 - s
    M = 0xFFFFFFFF
    r = random.Random(N * 31 + D)
    n3 = 3 * N
    for _ in range(3000):
        ra, rc = r.randrange(1 << (D - 4)), r.randrange(1 << (D - 4))
        i0, j0 = ra << 4, rc << 4
        ex, ey = r.randrange(N), r.randrange(N)
        alpha = (1 << D) - 2 * i0
        beta_m1 = (N << D) - n3 * j0 - 1
        G1 = ex * alpha + (ey << D) + beta_m1          # G(SW corner) - 1, exact (any sign)
        alpha_s = ((alpha & M) << k) & M
        ey_s = (1 << (D + k)) & M if D + k < 32 else 0
        beta_s = ((beta_m1 & M) << k) & M
        y0s = (ex * alpha_s + ey * ey_s + beta_s) & M
        assert y0s == (G1 << k) & M                    # so y0s = y0 2^k exactly when 0 <= y0 < 2^s
        y0 = r.randrange(16 * (2 * ex + n3))           # a line crossing the region
        assert y0 < (1 << s)
        assert ((((y0 << k) & M) * m) >> 32) == (y0 * m) >> s
        assert (((ex << (k + 1)) & M) * mlo) >> 32 == (2 * ex * mlo) >> s


def test_table_placement():
    """tab16_place / fill_tab16 / Raster16::boundary: for any 8-byte aligned table address S, the
    entries H + 256 (t + 2B) + 8 c (t in [-34, 56), c < 32) lie inside the array, B keeps every top
    byte f + B (f in [-17, 26]) inside 1..255, and X_u + X_(u+1) (one of them carrying H) is that
    address."""
    t_lo, n_tab, slots = -34, 90, (90 + 2) * 32
    r = random.Random(3)
    for _ in range(20000):
        S = r.randrange(0, 1 << 24) * 8 + (r.randrange(4) << 24)
        H = S & 0xFFFF0000
        two_b = ((S - H + 255) >> 8) - t_lo
        two_b += two_b & 1
        B = two_b >> 1
        assert 17 <= B <= 145
        first = H + 256 * (t_lo + 2 * B)
        assert S <= first and first + 256 * n_tab <= S + 8 * slots
        lane = r.randrange(32)
        f0 = r.randrange(-16, 27)
        f1 = f0 - r.randrange(2)
        lane_h = H | (4 * lane)
        x0 = ((f0 + B) << 8) | (lane_h & 0xFF) | (lane_h & 0xFFFF0000)   # even boundary: with H
        x1 = ((f1 + B) << 8) | (lane_h & 0xFF)                           # odd boundary
        assert 0 < f1 + B < 256 and x0 + x1 == first + 256 * (f0 + f1 - t_lo) + 8 * lane


@pytest.mark.parametrize("N", [1, 3, 64, 512, 8192, 32767])
def test_count_ahead_raster_matches_cell_tests(N):
    """k_pass count-ahead (chunk_math, CARaster): for a line crossing a parent of side 2^sh, the
    4-column raster on y' = (g - 1) >> (sh - 2) with the leaf fixed point marks exactly the 4x4
    grandchild cells (u, v) with 0 <= g - 1 - u Pg - v Qg < Pg + Qg (Pg = 2ex 2^(sh-2),
    Qg = 3N 2^(sh-2)): the paper's corner test at level l + 2."""
    s, m, mlo = fx_consts(N)
    n3 = 3 * N
    r = random.Random(11 + N)
    for _ in range(3000):
        sh = r.randrange(2, 16)
        ex = r.randrange(N)
        gm1 = r.randrange((1 << sh) * (2 * ex + n3))     # the line crosses the parent
        B = r.randrange(6, 135)
        y0 = gm1 >> (sh - 2)
        Y = ((y0 * m) >> s) + 1 + (B << 24)
        P = (2 * ex * mlo) >> s
        f = [(((Y - u * P) & 0xFFFFFFFF) >> 24) - B for u in range(5)]
        assert all(-5 <= x <= 6 for x in f)
        pg, qg = 2 * ex << (sh - 2), n3 << (sh - 2)
        for u in range(4):
            t = f[u] + f[u + 1]
            fu = (t + 1) // 2 if t >= 0 else -((-t) // 2)
            rows = set(range(max(t - fu, 0), min(fu, 3) + 1))
            direct = {v for v in range(4) if 0 <= gm1 - u * pg - v * qg < pg + qg}
            assert rows == direct, (N, sh, ex, gm1, u)


def _prmt(a, b, sel):
    bs = [(a >> (8 * i)) & 255 for i in range(4)] + [(b >> (8 * i)) & 255 for i in range(4)]
    return sum(bs[(sel >> (4 * k)) & 7] << (8 * k) for k in range(4))


def test_count_ahead_child_bits_gather():
    """k_pass MODE_WRITE derives the 4 child bits (NE, NW, SW, SE at bits 0..3) from the count-ahead
    raster's column words (byte v of word u = cell (u, v) crossed): a child is crossed iff one of its
    2x2 cells is (containment and the SW + NE identity). Exhaustive over the 2^16 cell patterns."""
    for pat in range(1 << 16):
        mc = [sum(((pat >> (4 * u + v)) & 1) << (8 * v) for v in range(4)) for u in range(4)]
        a, b = mc[0] | mc[1], mc[2] | mc[3]
        x = _prmt(a, b, 0x4026) | _prmt(a, b, 0x5137)
        nib = ((x * 0x10204080) & 0xFFFFFFFF) >> 28

        def anyc(da, dc):
            return int(any((pat >> (4 * (2 * da + i) + 2 * dc + j)) & 1 for i in (0, 1) for j in (0, 1)))
        assert nib == anyc(1, 1) | anyc(0, 1) << 1 | anyc(0, 0) << 2 | anyc(1, 0) << 3
