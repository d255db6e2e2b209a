"""Host model of k_edges16's packed 16-bit Sobel arithmetic (csrc/hht_kernels.cu edge_masks16)
against the plain 3x3 definition ("Sobel's gradient operator", R18-R21):
two pixels per 32-bit word with positive biases, |v| as a packed signed max, the edge and ALPHA
decisions as the top bit of each half. Checks the bias ranges (no borrow across halves) and the
column bookkeeping on random and extreme rows; the GPU kernel itself is compared with
oracle/frontend.py in tests/test_gpu_frontend.py."""
import numpy as np

M = 0xFFFFFFFF


def _bp(x, y, s):
    b = [(x >> (8 * i)) & 255 for i in range(4)] + [(y >> (8 * i)) & 255 for i in range(4)]
    return sum(b[(s >> (4 * i)) & 7] << (8 * i) for i in range(4))


def _vmaxs2(a, b):
    r = 0
    for h in (0, 16):
        x, y = (a >> h) & 0xFFFF, (b >> h) & 0xFFFF
        sx = x - 65536 if x >= 32768 else x
        sy = y - 65536 if y >= 32768 else y
        r |= (max(sx, sy) & 0xFFFF) << h
    return r


def packed(rows, hl, hr, thr, hasl, hasr):
    S, T = [0] * 8, [0] * 8
    for g in range(4):
        u, c, d = [int.from_bytes(bytes(rows[j][4 * g:4 * g + 4]), "little") for j in range(3)]
        ue, ce, de = u & 0xFF00FF, c & 0xFF00FF, d & 0xFF00FF
        uo, co, do = _bp(u, 0, 0x4341), _bp(c, 0, 0x4341), _bp(d, 0, 0x4341)
        S[2 * g], S[2 * g + 1] = (ue + 2 * ce + de) & M, (uo + 2 * co + do) & M
        T[2 * g], T[2 * g + 1] = (ue - de + 0x01000100) & M, (uo - do + 0x01000100) & M
    sl, sr = hl[0] + 2 * hl[1] + hl[2], hr[0] + 2 * hr[1] + hr[2]
    tl, tr = hl[0] - hl[2] + 256, hr[0] - hr[2] + 256
    E = Q = 0
    thr = min(thr, 2041)
    ke = (0x80008000 - 0x44004400 - thr * 0x10001) & M
    for g in range(4):
        Sl = _bp(sl, S[1], 0x5410) if g == 0 else _bp(S[2 * g - 1], S[2 * g + 1], 0x5432)
        Tl = _bp(tl, T[1], 0x5410) if g == 0 else _bp(T[2 * g - 1], T[2 * g + 1], 0x5432)
        Sr = _bp(S[6], sr, 0x5432) if g == 3 else _bp(S[2 * g], S[2 * g + 2], 0x5432)
        Tr = _bp(T[6], tr, 0x5432) if g == 3 else _bp(T[2 * g], T[2 * g + 2], 0x5432)
        for o in range(2):
            s_lo, s_hi = (Sl, S[2 * g + 1]) if o == 0 else (S[2 * g], Sr)
            t_lo, t_hi = (Tl, T[2 * g + 1]) if o == 0 else (T[2 * g], Tr)
            gxb = (s_hi - s_lo + 0x40004000) & M
            ax = _vmaxs2(gxb, (0x80008000 - gxb) & M)
            gyb = (t_lo + t_hi + 2 * T[2 * g + o]) & M
            ay = _vmaxs2(gyb, (0x08000800 - gyb) & M)
            e, q = (ax + ay + ke) & M, (ay - ax + 0xBC00BC00) & M
            sh = 15 - (4 * g + o)
            E |= (e >> sh) & (0x10001 << (4 * g + o))
            Q |= (q >> sh) & (0x10001 << (4 * g + o))
    em = (E | (E >> 14)) & 0xFFFF
    if not hasl:
        em &= ~1
    if not hasr:
        em &= ~0x8000
    return em, (Q | (Q >> 14)) & em


def plain(rows, hl, hr, thr, hasl, hasr):
    em = am = 0
    full = [[hl[j]] + list(rows[j]) + [hr[j]] for j in range(3)]
    for k in range(16):
        if (k == 0 and not hasl) or (k == 15 and not hasr):
            continue
        v = [[full[j][k + dx] for dx in range(3)] for j in range(3)]
        gx = (v[0][2] - v[0][0]) + 2 * (v[1][2] - v[1][0]) + (v[2][2] - v[2][0])
        gy = (v[0][0] + 2 * v[0][1] + v[0][2]) - (v[2][0] + 2 * v[2][1] + v[2][2])
        if abs(gx) + abs(gy) >= thr:
            em |= 1 << k
            if abs(gx) <= abs(gy):
                am |= 1 << k
    return em, am


def test_packed_sobel_matches_plain_definition():
    rng = np.random.default_rng(0)
    for it in range(4000):
        mode = it % 4
        if mode == 0:
            rows = rng.integers(0, 256, (3, 16))
        elif mode == 1:
            rows = rng.choice([0, 255], (3, 16))          # extreme gradients: |gx|, |gy| up to 1020
        elif mode == 2:
            rows = rng.integers(0, 4, (3, 16)) * 85
        else:
            rows = rng.choice([0, 1, 254, 255], (3, 16))
        hasl, hasr = bool(rng.integers(2)), bool(rng.integers(2))
        hl = [int(x) if hasl else 0 for x in rng.choice([0, 255, 128], 3)]
        hr = [int(x) if hasr else 0 for x in rng.choice([0, 255, 77], 3)]
        thr = int(rng.choice([1, 2, 50, 255, 256, 1000, 1020, 2040, 2041, 3000, 100000]))
        rows = [[int(x) for x in r] for r in rows]
        assert packed(rows, hl, hr, thr, hasl, hasr) == plain(rows, hl, hr, thr, hasl, hasr), (rows, hl, hr, thr)
