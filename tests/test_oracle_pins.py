"""Pins for the CPU oracle (oracle/hht_oracle.c) against things other than itself.

Each test names what fixes the expected value: a value printed in PAPER.md/SPEC.md (tests/golden),
a closed form, an invariant of the geometry, exact rational arithmetic, a brute force on tiny
inputs, or the independent survey enumeration. A plausible oracle mistake (a dropped term, a wrong
sign or index, a transposed operand, a wrong bit order, a non-strict threshold) fails at least one.
"""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------------------------------------
# Corner sign / code: printed examples
# ---------------------------------------------------------------------------------------------

def test_corner_sign_spec_examples():
    """SPEC.md:182-183 worked numerators (208 > 0 below; -240 on/above)."""
    for c in _gold("paper_spec_examples.json")["corner_sign"]["cases"]:
        assert oracle.corner_below(c["ex"], c["ey"], c["N"], c["D"], c["i"], c["j"]) == c["below"]


def test_lattice_code_spec_examples():
    """(0,3) at the root -> 0011; uniform 0000 / 1111 cases."""
    for c in _gold("paper_spec_examples.json")["lattice_code"]["cases"]:
        got = oracle.code(c["x"], c["y"], oracle.ALPHA, c["N"], c["D"], c["level"], c["a"], c["c"])
        assert got == c["code"], c


def test_fig2_generic_square_codes():
    """bit order NE,NW,SW,SE and 'above iff F >= 0'; row 1 is the paper's prose
    example for Fig. 2 line 1 (1011). A transposed bit order or a flipped convention fails."""
    for c in _gold("paper_spec_examples.json")["generic_square"]["cases"]:
        got = oracle.generic_code(c["m"][0], c["m"][1], c["b"][0], c["b"][1], 0, 0, 1)
        assert format(got, "04b") == c["code"], c["line"]
        assert (got not in (0, 15)) == c["votes"]


def test_code_1101_unrealizable():
    """DESIGN.md R3: SW above with NW below would need b <= 0 and b > 1 on the unit square, so the
    paper's listed '1, 1, 0, 1' for Fig. 2 line 1 cannot occur for any non-vertical line."""
    seen = set()
    for mn in range(-40, 41):
        for bn in range(-40, 41):
            seen.add(oracle.generic_code(mn, 8, bn, 8, 0, 0, 1))
    assert 0b1101 not in seen
    assert {0b1011, 0b0011, 0b0001, 0b0111, 0, 15} <= seen


# ---------------------------------------------------------------------------------------------
# Corner sign: exact rationals
# ---------------------------------------------------------------------------------------------

def test_corner_sign_matches_exact_rationals():
    """the int64 fixed-point sign equals the exact rational sign of
    y0 - x0*m_c - b_c with m_c = -1 + 2i/2^D, b_c = -N + 3N*j/2^D (root [-1,1] x [-N,2N])."""
    rng = random.Random(1234)
    for _ in range(20000):
        D = rng.randint(1, 14)
        N = rng.randint(1, 5000)
        ex, ey = rng.randrange(N), rng.randrange(N)
        i, j = rng.randint(0, 1 << D), rng.randint(0, 1 << D)
        m_c = Fraction(-1) + Fraction(2 * i, 1 << D)
        b_c = Fraction(-N) + Fraction(3 * N * j, 1 << D)
        below = b_c < ey - ex * m_c                     # corner strictly below b = ey - ex*m
        assert oracle.corner_below(ex, ey, N, D, i, j) == int(below), (ex, ey, N, D, i, j)


def test_beta_half_swaps_coordinates():
    """a BETA point (x0,y0) is treated as (y0,x0)."""
    rng = random.Random(7)
    for _ in range(3000):
        D = rng.randint(1, 6)
        N = rng.randint(2, 40)
        x, y = rng.randrange(N), rng.randrange(N)
        lev = rng.randint(0, D)
        a, c = rng.randrange(1 << lev), rng.randrange(1 << lev)
        assert oracle.code(x, y, oracle.BETA, N, D, lev, a, c) == oracle.code(y, x, oracle.ALPHA, N, D, lev, a, c)


# ---------------------------------------------------------------------------------------------
# Closed forms
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("N,D", [(5, 2), (8, 3), (16, 4), (12, 5)])
def test_horizontal_parameter_line_closed_form(N, D):
    """A point (0, y) maps to the constant line b = y. A region [m0,m1] x [b0,b1] then has its two
    lower corners below iff b0 < y and its two upper corners below iff b1 < y, so it votes iff
    b0 < y <= b1: exactly one row of regions per level, every column. Checked for every y, level
    and region with exact rationals (catches a<->c transposition and sign slips)."""
    for y in range(N):
        pts = np.array([[0, y]], dtype=np.int32)
        for lev in range(D + 1):
            acc = oracle.dense_votes(pts, oracle.ALPHA, N, D, lev)     # acc[c, a]
            side = 1 << lev
            for c in range(side):
                b0 = Fraction(-N) + Fraction(3 * N * c, side)
                b1 = Fraction(-N) + Fraction(3 * N * (c + 1), side)
                want = 1 if (b0 < y <= b1) else 0
                assert (acc[c] == want).all(), (y, lev, c)


def _raster_leaf_votes(points, N, D):
    """The classic slope-intercept accumulator by walking each line across the m-axis columns
    (SPEC.md:316-324): in column [m_a, m_a+1] the line b(m) = ey - ex*m spans [b(m_a+1), b(m_a)]
    (ex >= 0). A cell [B_c, B_c+1] has some corner strictly below the line iff B_c < b(m_a), and
    some corner on/above iff B_c+1 >= b(m_a+1); it votes iff both."""
    side = 1 << D
    acc = np.zeros((side, side), dtype=np.int64)
    for ex, ey in points:
        for a in range(side):
            mL = Fraction(-1) + Fraction(2 * a, side)
            mR = Fraction(-1) + Fraction(2 * (a + 1), side)
            bL, bR = ey - ex * mL, ey - ex * mR
            for c in range(side):
                B0 = Fraction(-N) + Fraction(3 * N * c, side)
                B1 = Fraction(-N) + Fraction(3 * N * (c + 1), side)
                if B0 < bL and B1 >= bR:
                    acc[c, a] += 1
    return acc


@pytest.mark.parametrize("seed", range(6))
def test_leaf_accumulator_equals_rasterisation(seed):
    rng = random.Random(seed)
    N = rng.choice([4, 6, 8, 11])
    D = rng.choice([2, 3])
    pts = [(rng.randrange(N), rng.randrange(N)) for _ in range(rng.randint(1, 12))]
    got = oracle.dense_votes(np.array(pts, dtype=np.int32), oracle.ALPHA, N, D, D)
    assert (got.astype(np.int64) == _raster_leaf_votes(pts, N, D)).all()


@pytest.mark.parametrize("N,D", [(5, 2), (6, 3), (8, 3), (16, 4), (8, 5)])
def test_realizable_codes_only(N, D):
    """with 0 <= ex < N every region has G_SW >= G_SE > G_NW >= G_NE, so the
    only codes are 0000, 0010, 0011, 0111, 1111; 0000/1111 never vote."""
    seen = set()
    for ex in range(N):
        for ey in range(N):
            for lev in range(D + 1):
                for a in range(1 << lev):
                    for c in range(1 << lev):
                        seen.add(oracle.code(ex, ey, oracle.ALPHA, N, D, lev, a, c))
    assert seen <= {0b0000, 0b0010, 0b0011, 0b0111, 0b1111}
    assert {0b0010, 0b0011, 0b0111} <= seen


# ---------------------------------------------------------------------------------------------
# The independent survey enumeration
# ---------------------------------------------------------------------------------------------

def test_survey_worked_example():
    """SURVEY.md §8(c) item 5 (tests/golden/survey_example_n8_d3_t2.json): records per level in DFS
    quad order NE,NW,SW,SE, leaves, total votes and tests."""
    g = _gold("survey_example_n8_d3_t2.json")
    r = oracle.detect(g["points"], g["N"], g["D"], g["T"], halves=g["halves"])
    for lev, recs in g["levels"].items():
        assert r.levels[(oracle.ALPHA, int(lev))].tolist() == recs, lev
    assert r.leaves[:, 1:].tolist() == g["leaves"]
    assert r.votes == g["votes"] and r.tests == g["tests"]
    # true line y = x -> (m, b) = (1, 0) lies in leaf (7, 2): m in [0.75, 1], b in [-2, 1]
    assert [7, 2, 4] in g["leaves"]


# ---------------------------------------------------------------------------------------------
# Invariants and brute force on random tiny scenes
# ---------------------------------------------------------------------------------------------

_QUAD = [(1, 1), (0, 1), (0, 0), (1, 0)]   # NE, NW, SW, SE


def _check_tree(pts, N, D, T, half, r):
    E = pts.shape[0]
    dense = [oracle.dense_votes(pts, half, N, D, lev) for lev in range(D + 1)]
    recs = [r.levels[(half, lev)] for lev in range(D + 1)]
    # root = E (L7: every line crosses the root)
    assert recs[0].tolist() == [[0, 0, E]]
    # votes(R) for every visited R = brute force over ALL points (L5: restriction loses nothing)
    for lev in range(D + 1):
        for a, c, v in recs[lev].tolist():
            assert dense[lev][c, a] == v, (lev, a, c)
    # visited set: children (in quad order) of every visited region with votes > T, nothing else
    expect = [[(0, 0)]]
    for lev in range(D):
        nxt = []
        for a, c, v in recs[lev].tolist():
            if v > T:
                nxt += [(2 * a + da, 2 * c + dc) for da, dc in _QUAD]
        expect.append(nxt)
    for lev in range(D + 1):
        assert [(a, c) for a, c, _ in recs[lev].tolist()] == expect[lev]
    # child <= parent; parent <= sum(children) <= 3 * parent (L5, L6)
    for lev in range(D):
        kids = iter(recs[lev + 1].tolist())
        for a, c, v in recs[lev].tolist():
            if v > T:
                ch = [next(kids)[2] for _ in range(4)]
                assert max(ch) <= v
                assert v <= sum(ch) <= 3 * v
                # G_SW >= G_centre >= G_NE: a line crosses R iff it crosses exactly one of R's SW
                # child (G_SW > 0 >= G_centre) and NE child (G_centre > 0 >= G_NE)
                assert v == ch[2] + ch[0]
    # leaves = {leaf : brute votes > T} (removal off)
    leaves = {(int(i), int(j)) for h, i, j, _ in r.leaves.tolist() if h == half}
    brute = {(a, c) for c, a in zip(*np.nonzero(dense[D] > T))}
    assert leaves == brute


@pytest.mark.parametrize("seed", range(60))
def test_oracle_tree_invariants_random(seed):
    rng = random.Random(seed)
    N = rng.choice([4, 5, 8, 13, 16, 32])
    D = rng.choice([1, 2, 3, 4, 5]) if N >= 8 else rng.choice([1, 2, 3])
    T = rng.choice([1, 2, 5, 20])
    pts = synth.random_scene(seed, N, max_lines=3, max_noise=80)
    r = oracle.detect(pts, N, D, T, halves=oracle.ALPHA | oracle.BETA)
    for half in (oracle.ALPHA, oracle.BETA):
        _check_tree(pts, N, D, T, half, r)
    # tests = E per tree at the root + 4 * votes of every split region (R9)
    E = pts.shape[0]
    want = 0
    for half in (oracle.ALPHA, oracle.BETA):
        want += E
        for lev in range(D):
            want += 4 * sum(v for _, _, v in r.levels[(half, lev)].tolist() if v > T)
    assert r.tests == want
    assert r.votes == sum(int(v[:, 2].sum()) for v in r.levels.values())


def test_threshold_is_strict():
    """PAPER.md:122 'if level.vote > THRESHOLD': a region with exactly T votes does not split."""
    pts = np.array([[0, 3]] * 5, dtype=np.int32)
    r = oracle.detect(pts, 8, 3, 5, halves=oracle.ALPHA)
    assert r.levels[(oracle.ALPHA, 0)].tolist() == [[0, 0, 5]]
    assert r.levels[(oracle.ALPHA, 1)].shape[0] == 0
    r = oracle.detect(pts, 8, 3, 4, halves=oracle.ALPHA)
    assert r.levels[(oracle.ALPHA, 1)].shape[0] == 4


def test_empty_input():
    r = oracle.detect(np.zeros((0, 2), np.int32), 8, 3, 1)
    assert r.levels[(oracle.ALPHA, 0)].tolist() == [[0, 0, 0]]
    assert r.leaves.shape[0] == 0 and r.votes == 0 and r.tests == 0


# ---------------------------------------------------------------------------------------------
# FHT circumcircle variant (north_star "FHT casts extra false votes")
# ---------------------------------------------------------------------------------------------

def test_circle_contains_exact_everywhere():
    """Exact crossing implies within the circumradius: per (point, region)."""
    for N, D in [(8, 3), (16, 4), (6, 3)]:
        for ex in range(N):
            for ey in range(N):
                for lev in range(D + 1):
                    for a in range(1 << lev):
                        for c in range(1 << lev):
                            if oracle.code(ex, ey, oracle.ALPHA, N, D, lev, a, c) not in (0, 15):
                                assert oracle.circle_passes(ex, ey, oracle.ALPHA, N, D, lev, a, c)


def test_category2_line_exists():
    """PAPER.md:33 Fig. 1 line 2: inside the circumcircle but not through the square."""
    N, D = 16, 4
    found = False
    for ex in range(N):
        for ey in range(N):
            for a in range(4):
                for c in range(4):
                    if oracle.circle_passes(ex, ey, oracle.ALPHA, N, D, 2, a, c) and \
                            oracle.code(ex, ey, oracle.ALPHA, N, D, 2, a, c) in (0, 15):
                        found = True
    assert found


@pytest.mark.parametrize("cid", [1, 2])
def test_circle_variant_casts_extra_votes(cid):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    ex = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves, variant=0)
    ci = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves, variant=1)
    assert ci.votes > ex.votes
    # node-wise domination on the nodes both variants visit
    for key, recs in ex.levels.items():
        cmap = {(a, c): v for a, c, v in ci.levels[key].tolist()}
        for a, c, v in recs.tolist()[:2000]:
            if (a, c) in cmap:
                assert cmap[(a, c)] >= v


# ---------------------------------------------------------------------------------------------
# Synthetic recovery
# ---------------------------------------------------------------------------------------------

def test_c1_recovers_generated_lines():
    """Each generated C1 line's (m, b) lies in or next to an emitted leaf cell
    (cell widths 2/2^D in m and 3N/2^D in b, PAPER.md:69 reading R10)."""
    cfg = synth.CONFIGS[1]
    pts, truth = synth.config_image(1)
    r = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    side = 1 << cfg.D
    cells = {(int(i), int(j)) for _, i, j, _ in r.leaves.tolist()}
    assert cells
    for t in truth:
        m = Fraction(t.A, 1 << 16)
        b = Fraction(t.Q, 1 << 16)
        i = int((m + 1) * side / 2)
        j = int((b + cfg.N) * side / (3 * cfg.N))
        near = {(i + di, j + dj) for di in (-1, 0, 1) for dj in (-1, 0, 1)}
        assert near & cells, (t, i, j)


# ---------------------------------------------------------------------------------------------
# The circumcircle tests pinned to geometry computed another way ("calculates the
# perpendicular distance to the line from the center of the region and compares it with the radius
# of the circle circumscribing the region"). The oracle squares the point-line distance formula;
# here the squared distance is the minimum over the line of the squared distance to the centre,
# found by setting the derivative of a quadratic to zero, in exact rationals.
# ---------------------------------------------------------------------------------------------

def _min_sq_dist_lattice(ex, ey, N, D, i_c, j_c):
    """min over points (i, j) of the lattice line 2ex*i + 3N*j = 2^D (ex+ey+N) of (i-i_c)^2 + (j-j_c)^2."""
    K = Fraction((1 << D) * (ex + ey + N), 3 * N)
    k = Fraction(2 * ex, 3 * N)                          # j(i) = K - k*i
    i = (i_c + k * (K - j_c)) / (1 + k * k)              # d/di [(i-i_c)^2 + (K-k*i-j_c)^2] = 0
    return (i - i_c) ** 2 + (K - k * i - j_c) ** 2


def _min_sq_dist_mb(ex, ey, m_c, b_c):
    """min over m of (m-m_c)^2 + (ey - ex*m - b_c)^2 (points (m, b) of the line b = ey - ex*m)."""
    m = (m_c + ex * (ey - b_c)) / (1 + ex * ex)
    return (m - m_c) ** 2 + (ey - ex * m - b_c) ** 2


@pytest.mark.parametrize("N,D", [(5, 2), (8, 3), (16, 4), (6, 4)])
def test_circle_lattice_units_matches_minimised_distance(N, D):
    """Variant 1: the line meets the circle through the 4 corners of the s x s lattice square
    (radius s/sqrt(2), centre (i0 + s/2, j0 + s/2)) iff its minimum squared distance <= s^2/2."""
    rng = random.Random(N * 100 + D)
    pts = [(x, y) for x in range(N) for y in range(N)]
    if len(pts) > 80:
        pts = rng.sample(pts, 80)
    for x, y in pts:
        for half in (oracle.ALPHA, oracle.BETA):
            ex, ey = (x, y) if half == oracle.ALPHA else (y, x)
            for lev in range(D + 1):
                s = 1 << (D - lev)
                for a in range(1 << lev):
                    for c in range(1 << lev):
                        d2 = _min_sq_dist_lattice(ex, ey, N, D, Fraction(2 * a * s + s, 2), Fraction(2 * c * s + s, 2))
                        want = int(d2 <= Fraction(s * s, 2))
                        assert oracle.circle_passes(x, y, half, N, D, lev, a, c) == want, (x, y, half, lev, a, c)


def test_circle_lattice_units_horizontal_closed_form():
    """ex = 0: the parameter line is horizontal, b = ey, i.e. lattice row j* = 2^D (ey+N)/(3N); the
    circle of radius s/sqrt(2) around (., j_c) meets it iff 2 (j_c - j*)^2 <= s^2."""
    for N, D in [(8, 3), (16, 4), (12, 5)]:
        for ey in range(N):
            jstar = Fraction((1 << D) * (ey + N), 3 * N)
            for lev in range(D + 1):
                s = 1 << (D - lev)
                for c in range(1 << lev):
                    jc = Fraction(2 * c * s + s, 2)
                    want = int(2 * (jc - jstar) ** 2 <= s * s)
                    for a in (0, (1 << lev) - 1):
                        assert oracle.circle_passes(0, ey, oracle.ALPHA, N, D, lev, a, c) == want


def test_circle_survey_l9_totals():
    """SURVEY.md §0 L9 (the survey's independent enumeration): N=16, D=4 over all effective points
    and all regions of all levels: 10,356 exact votes, 1,554 extra circle votes."""
    g = _gold("survey_l9_circle_n16_d4.json")
    N, D = g["N"], g["D"]
    exact = extra = 0
    for x in range(N):
        for y in range(N):
            for lev in range(D + 1):
                for a in range(1 << lev):
                    for c in range(1 << lev):
                        e = oracle.code(x, y, oracle.ALPHA, N, D, lev, a, c) not in (0, 15)
                        p = oracle.circle_passes(x, y, oracle.ALPHA, N, D, lev, a, c)
                        assert p or not e
                        exact += e
                        extra += p and not e
    assert (exact, extra) == (g["exact_votes"], g["extra_circle_votes"])


@pytest.mark.parametrize("N,D", [(5, 2), (8, 3), (16, 4), (6, 4)])
def test_circle_mb_units_matches_minimised_distance(N, D):
    """Variant 2 (reading R22): the region is the rectangle [m0, m0 + 2s/2^D] x [b0, b0 + 3Ns/2^D]
    with m0 = -1 + 2 i0/2^D, b0 = -N + 3N j0/2^D; its circumcircle has the centre of the rectangle
    and radius^2 = (w^2 + h^2)/4; the line b = ey - ex*m meets it iff min squared distance <= radius^2."""
    rng = random.Random(N * 1000 + D)
    pts = [(x, y) for x in range(N) for y in range(N)]
    if len(pts) > 80:
        pts = rng.sample(pts, 80)
    S = 1 << D
    for x, y in pts:
        for half in (oracle.ALPHA, oracle.BETA):
            ex, ey = (x, y) if half == oracle.ALPHA else (y, x)
            for lev in range(D + 1):
                s = 1 << (D - lev)
                w, h = Fraction(2 * s, S), Fraction(3 * N * s, S)
                for a in range(1 << lev):
                    for c in range(1 << lev):
                        m_c = -1 + Fraction(2 * a * s, S) + w / 2
                        b_c = -N + Fraction(3 * N * c * s, S) + h / 2
                        want = int(_min_sq_dist_mb(ex, ey, m_c, b_c) <= (w * w + h * h) / 4)
                        assert oracle.circle_mb_passes(x, y, half, N, D, lev, a, c) == want, (x, y, half, lev, a, c)


@pytest.mark.parametrize("passes", ["circle_passes", "circle_mb_passes"])
def test_circle_variants_contain_exact_and_nest(passes):
    """Both circle tests accept every exactly-crossing line (the circle contains the region), and a
    child's circumcircle lies inside its parent's (radius halves, centre moves by half the parent's
    radius), so passing a child implies passing the parent: the candidate-list restriction of
    PAPER.md:100-103 stays exact for both variants."""
    f = getattr(oracle, passes)
    for N, D in [(8, 3), (16, 4), (7, 3)]:
        for ex in range(N):
            for ey in range(N):
                for lev in range(D + 1):
                    for a in range(1 << lev):
                        for c in range(1 << lev):
                            p = f(ex, ey, oracle.ALPHA, N, D, lev, a, c)
                            if oracle.code(ex, ey, oracle.ALPHA, N, D, lev, a, c) not in (0, 15):
                                assert p
                            if p and lev > 0:
                                assert f(ex, ey, oracle.ALPHA, N, D, lev - 1, a >> 1, c >> 1)


def test_circle_mb_reading_grows_with_size():
    """Reading R22's qualitative consequence (Table 1 C_v grows with the image size):
    in (m, b) units the circumcircle is wide compared with the region for steep parameter lines,
    so the extra votes per exact vote grow with N on uniform scenes (strictly, for N = 8, 16, 32)."""
    ratios = []
    for N in (8, 16, 32):
        D = N.bit_length() - 1
        rng = np.random.default_rng(N)
        pts = rng.integers(0, N, size=(3 * N, 2)).astype(np.int32)
        ex_ = oracle.detect(pts, N, D, 1 << 30, oracle.ALPHA, variant=0)
        tot_e = tot_c = 0
        for lev in range(D + 1):
            for a in range(1 << lev):
                for c in range(1 << lev):
                    tot_e += oracle.region_votes(pts, oracle.ALPHA, N, D, lev, a, c, 0)
                    tot_c += oracle.region_votes(pts, oracle.ALPHA, N, D, lev, a, c, 2)
        assert ex_.votes == pts.shape[0]
        ratios.append(tot_c / tot_e)
    assert ratios[0] < ratios[1] < ratios[2], ratios
