"""Pins of the oracle's edge front end (oracle/frontend.py; §3, readings DESIGN.md
R18-R21 after SPEC.md:104-131): SPEC's worked examples, the convolution against a library routine
(scipy.ndimage.correlate on the interior), and the partition invariants."""
import numpy as np
import pytest
from scipy import ndimage

import oracle


def test_constant_image_has_no_gradient():
    gx, gy = oracle.sobel(np.full((9, 7), 77, np.uint8))
    assert not gx.any() and not gy.any()
    a, b = oracle.edges(np.full((9, 7), 77, np.uint8), 1)
    assert a.shape == (0, 2) and b.shape == (0, 2)


def test_vertical_step_is_beta():
    img = np.zeros((8, 10), np.uint8)
    img[:, 5:] = 255
    gx, gy = oracle.sobel(img)
    assert (np.abs(gx[1:-1, 4:6]) == 4 * 255).all() and not gy.any()
    a, b = oracle.edges(img, 128)
    assert a.shape[0] == 0 and b.shape[0] == 2 * 6
    assert set(map(tuple, b.tolist())) == {(x, y) for x in (4, 5) for y in range(1, 7)}


def test_horizontal_step_is_alpha():
    img = np.zeros((8, 10), np.uint8)
    img[:4, :] = 255                                                     # top half bright
    gx, gy = oracle.sobel(img)
    assert not gx.any() and (gy[3:5, 1:-1] == 4 * 255).all()             # SPEC.md:113; brighter above: gy > 0
    a, b = oracle.edges(img, 128)
    assert b.shape[0] == 0 and a.shape[0] == 2 * 8
    # raster order: row 3 (y = 4) before row 4 (y = 3), columns ascending
    assert a.tolist() == [[x, 4] for x in range(1, 9)] + [[x, 3] for x in range(1, 9)]


def test_tie_goes_to_alpha():
    """|gx| = |gy| != 0 -> ALPHA (slope bound inclusive): a symmetric diagonal edge."""
    n = 9
    r, c = np.mgrid[0:n, 0:n]
    img = np.where(c + (n - 1 - r) >= n, 255, 0).astype(np.uint8)     # bright where x + y >= n
    gx, gy = oracle.sobel(img)
    on = (gx != 0) | (gy != 0)
    assert on.any() and (np.abs(gx[on]) == np.abs(gy[on])).all()
    a, b = oracle.edges(img, 1)
    assert b.shape[0] == 0 and a.shape[0] == int(on.sum())


@pytest.mark.parametrize("seed", range(5))
def test_sobel_matches_library_correlation(seed):
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=(13, 17), dtype=np.uint8)
    gx, gy = oracle.sobel(img)
    I = img.astype(np.int64)
    kx = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]])
    ky = np.array([[1, 2, 1], [0, 0, 0], [-1, -2, -1]])      # row above (geometric y+1) positive
    cx = ndimage.correlate(I, kx, mode="constant")[1:-1, 1:-1]
    cy = ndimage.correlate(I, ky, mode="constant")[1:-1, 1:-1]
    assert np.array_equal(gx[1:-1, 1:-1], cx) and np.array_equal(gy[1:-1, 1:-1], cy)
    assert not gx[[0, -1], :].any() and not gx[:, [0, -1]].any()   # border gradients are zero
    assert not gy[[0, -1], :].any() and not gy[:, [0, -1]].any()


@pytest.mark.parametrize("seed", range(5))
def test_partition_invariants(seed):
    rng = np.random.default_rng(100 + seed)
    img = rng.integers(0, 256, size=(16, 16), dtype=np.uint8)
    gx, gy = oracle.sobel(img)
    prev = None
    for thr in (0, 1, 200, 600, 2000):
        a, b = oracle.partition_edges(gx, gy, thr)
        pts = set(map(tuple, a.tolist())) | set(map(tuple, b.tolist()))
        assert len(pts) == a.shape[0] + b.shape[0]                     # each edge point in one set
        for x, y in a.tolist():
            r = 15 - y
            assert abs(gx[r, x]) <= abs(gy[r, x]) and abs(gx[r, x]) + abs(gy[r, x]) >= thr
        for x, y in b.tolist():
            r = 15 - y
            assert abs(gx[r, x]) > abs(gy[r, x]) and abs(gx[r, x]) + abs(gy[r, x]) >= thr
        if thr == 0:
            assert not pts                                              # thr > 0
        if prev is not None and thr > 0:
            assert pts <= prev                                          # monotone shrinkage
        prev = pts if thr > 0 else None
        if thr > 0:
            rows = [(15 - y, x) for x, y in a.tolist()]
            assert rows == sorted(rows)                                 # raster order
