"""GPU edge front end against the oracle's front end
(oracle/frontend.py, pinned in tests/test_frontend_oracle.py): the ALPHA and BETA edge lists must be
identical (same points, same raster order), and hht_detect_image / hht_detect_trees must give the
oracle's records, leaves and statistics with the ALPHA tree run on the ALPHA points only and the BETA
tree on the BETA points only."""
import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import compare_tree

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


def line_image(N, seed, lines=4, noise=0.01):
    """Synthetic grayscale image: line pixels (from the seeded generator) at 255 over a dark
    background with sparse salt noise; row 0 = top, pixel (x, y) at row N-1-y."""
    pts, _ = synth.scene(N, lines, max(2, N // 2), 1 if N > 8 else 0, int(noise * N * N), False, 0xED6E, seed, 7)
    img = np.zeros((N, N), np.uint8)
    img[N - 1 - pts[:, 1], pts[:, 0]] = 255
    return img


def _images():
    rng = np.random.default_rng(5)
    out = []
    for N in (3, 4, 5, 17, 33, 64, 100, 129):
        out.append((f"random{N}", rng.integers(0, 256, size=(N, N), dtype=np.uint8), 300))
    for N, s in ((32, 1), (64, 2), (128, 3), (256, 4), (300, 5)):
        out.append((f"lines{N}", line_image(N, s), 255))
    step = np.zeros((40, 40), np.uint8)
    step[:, 20:] = 200
    out.append(("vstep", step, 100))
    out.append(("hstep", step.T.copy(), 100))
    out.append(("const", np.full((20, 20), 9, np.uint8), 1))
    return out


@pytest.mark.parametrize("name,img,thr", _images(), ids=[x[0] for x in _images()])
def test_edges_match_oracle(name, img, thr, cuda_device):
    import torch
    N = img.shape[0]
    a_ref, b_ref = oracle.edges(img, thr)
    h = hht.HHT(halves=AB)
    D = max(1, int(np.log2(N)))
    h.detect_image(torch.from_numpy(img).to(cuda_device), thr, D, 2)
    a, b = h.edges()
    assert np.array_equal(a, a_ref) and np.array_equal(b, b_ref), (a.shape, a_ref.shape, b.shape, b_ref.shape)


@pytest.mark.parametrize("N,kind", [(1040, "random"), (2048, "random"), (2048, "sparse")])
def test_edges_many_tiles(N, kind, cuda_device):
    """Widths that are a multiple of 16 with several super-tiles of 128 tiles (k_edges16_write sums
    the earlier super-tiles and tiles itself): 1040^2 = 265 tiles (a width that is not a power of two),
    2048^2 = 1024 tiles (8 super-tiles); dense random edges and a sparse image whose first super-tiles
    are empty. The threshold is above the point count, so the trees stop at the root."""
    import torch
    rng = np.random.default_rng(N)
    if kind == "random":
        img, thr = rng.integers(0, 256, size=(N, N), dtype=np.uint8), 300
    else:
        img, thr = np.zeros((N, N), np.uint8), 200
        img[N // 2 + 5, 7:N - 9:3] = 255
        img[N - 40:N - 2, N - 33] = 250
    a_ref, b_ref = oracle.edges(img, thr)
    assert a_ref.shape[0] + b_ref.shape[0] > 0
    h = hht.HHT(halves=AB)
    h.detect_image(torch.from_numpy(img).to(cuda_device), thr, 3, N * N)
    a, b = h.edges()
    assert np.array_equal(a, a_ref) and np.array_equal(b, b_ref), (a.shape, a_ref.shape, b.shape, b_ref.shape)


@pytest.mark.parametrize("N,seed,T", [(32, 11, 3), (64, 12, 6), (128, 13, 10), (256, 14, 24)])
def test_detect_image_matches_oracle(N, seed, T, cuda_device):
    import torch
    img = line_image(N, seed)
    thr, D = 255, int(np.log2(N))
    a_ref, b_ref = oracle.edges(img, thr)
    ra = oracle.detect(a_ref, N, D, T, hht.ALPHA)
    rb = oracle.detect(b_ref, N, D, T, hht.BETA)
    for src in ("device", "host"):
        h = hht.HHT(halves=AB)
        h.detect_image(torch.from_numpy(img).to(cuda_device) if src == "device" else img, thr, D, T)
        compare_tree(h, ra, 0, hht.ALPHA, D)
        compare_tree(h, rb, 0, hht.BETA, D)
        st = h.stats()
        assert (st["tests"], st["votes"]) == (ra.tests + rb.tests, ra.votes + rb.votes)
    # one half only: that half's points
    ha = hht.HHT(halves=hht.BETA)
    ha.detect_image(img, thr, D, T)
    compare_tree(ha, rb, 0, hht.BETA, D)
    assert ha.edges()[0].shape[0] == 0 and np.array_equal(ha.edges()[1], b_ref)


def test_detect_trees_batch(cuda_device):
    """Per-tree point sets over a batch: tree (b, ALPHA) and (b, BETA) get different points."""
    N, D, T = 64, 6, 4
    sets, offs = [], [0]
    for b in range(3):
        for half in (hht.ALPHA, hht.BETA):
            p = synth.random_scene(700 + 2 * b + half, N, max_lines=3, max_noise=150)
            sets.append(p)
            offs.append(offs[-1] + len(p))
    sets[3] = sets[3][:0]                                   # an empty tree
    offs = [0] + list(np.cumsum([len(p) for p in sets]))
    h = hht.HHT(halves=AB)
    h.detect_trees(np.concatenate(sets).astype(np.int32), offs, N, D, T)
    tests = 0
    for t, p in enumerate(sets):
        half = hht.ALPHA if t % 2 == 0 else hht.BETA
        ref = oracle.detect(p, N, D, T, half)
        compare_tree(h, ref, t // 2, half, D)
        tests += ref.tests
    assert h.stats()["tests"] == tests


def test_zero_threshold_has_no_edges(cuda_device):
    h = hht.HHT(halves=AB)
    h.detect_image(line_image(32, 1), 0, 5, 2)
    a, b = h.edges()
    assert a.shape[0] == 0 and b.shape[0] == 0 and h.stats()["leaves"] == 0
