"""Helpers shared by the parity tests: compare a libhht result with an oracle result, and check
structural invariants of a (possibly huge) libhht result with numpy."""
import numpy as np

QUAD = [(1, 1), (0, 1), (0, 0), (1, 0)]   # NE, NW, SW, SE


def compare_tree(h, ref, image, half, D, ref_image=0):
    """Bit-exact comparison of every level's (a, c, votes) records and the leaves of one tree."""
    for lev in range(D + 1):
        got = h.level(image, half, lev)
        want = ref.levels[(half, lev)]
        assert got.shape == want.shape, f"image {image} half {half} level {lev}: {got.shape} vs {want.shape}"
        if not np.array_equal(got, want):
            bad = np.nonzero((got != want).any(axis=1))[0][:5]
            raise AssertionError(f"image {image} half {half} level {lev}: first diffs at {bad}: "
                                 f"{got[bad].tolist()} vs {want[bad].tolist()}")
    lv = h.leaves(image)
    lv = lv[lv[:, 1] == half][:, 2:]
    want = ref.leaves[ref.leaves[:, 0] == half][:, 1:].astype(np.int64)
    assert np.array_equal(lv, want), f"image {image} half {half}: leaves differ ({len(lv)} vs {len(want)})"


def compare_all(h, ref, halves, D, image=0):
    for half in (1, 2):
        if halves & half:
            compare_tree(h, ref, image, half, D)


def check_structure(levels, E, T, D):
    """levels[l] = uint32 [k, 3] records (a, c, votes) of one tree in depth-first order. Checks:
    root = E; the visited set at l+1 is exactly the children (NE,NW,SW,SE) of the regions at l with
    votes > T, in order; child <= parent; parent <= sum(children) <= 3*parent;
    votes(parent) = votes(SW child) + votes(NE child).
    Returns (tests, votes) recomputed from the records."""
    assert levels[0].tolist() == [[0, 0, E]]
    tests, votes = E, int(levels[0][:, 2].sum())
    for lev in range(D):
        P = levels[lev].astype(np.int64)
        Cn = levels[lev + 1].astype(np.int64)
        split = P[:, 2] > T
        Ps = P[split]
        assert Cn.shape[0] == 4 * Ps.shape[0], (lev, Cn.shape, Ps.shape)
        if Ps.shape[0] == 0:
            continue
        ca = (2 * Ps[:, 0:1] + np.array([q[0] for q in QUAD])[None, :]).reshape(-1)
        cc = (2 * Ps[:, 1:2] + np.array([q[1] for q in QUAD])[None, :]).reshape(-1)
        assert np.array_equal(Cn[:, 0], ca) and np.array_equal(Cn[:, 1], cc), f"level {lev + 1} keys"
        cv = Cn[:, 2].reshape(-1, 4)
        assert (cv.max(axis=1) <= Ps[:, 2]).all(), f"child > parent at level {lev + 1}"
        s = cv.sum(axis=1)
        assert (s >= Ps[:, 2]).all() and (s <= 3 * Ps[:, 2]).all(), f"sum of children at level {lev + 1}"
        assert np.array_equal(cv[:, 0] + cv[:, 2], Ps[:, 2]), f"votes != SW + NE at level {lev}"
        tests += 4 * int(Ps[:, 2].sum())
        votes += int(Cn[:, 2].sum())
    return tests, votes
