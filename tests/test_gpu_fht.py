"""GPU parity of the FHT circumcircle variant: the same
level-synchronous pipeline with the membership test "the line meets the region's circumscribing
circle", compared bit-exactly with the oracle's variants 1 (circle in lattice units,
oracle_circle_passes) and 2 (circle in (m, b) units, oracle_circle_mb_passes; reading R22), both
pinned in tests/test_oracle_pins.py, plus the paper's claim that the circle test casts extra
(false) votes: at every region both runs visit, circle votes >= exact votes."""
import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import compare_all

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


def _dev(pts, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(pts, dtype=np.int32)).to(dev)


VARS = [hht.FHT_CIRCLE, hht.FHT_CIRCLE_MB]


def _run(pts, N, D, T, halves, dev, var=hht.FHT_CIRCLE, **kw):
    h = hht.HHT(halves=halves, variant=var, **kw)
    h.detect(_dev(pts, dev), N, D, T)
    return h


# variant 2 on config 2 costs the oracle ~3 min (9.3e9 tests: the (m, b) circle accepts far more)
CFG_VARS = [(1, hht.FHT_CIRCLE), (2, hht.FHT_CIRCLE), (1, hht.FHT_CIRCLE_MB)]


@pytest.mark.parametrize("cid,var", CFG_VARS)
def test_config_parity_circle(cid, var, cuda_device):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves, variant=var)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, cuda_device, var)
    compare_all(h, ref, cfg.halves, cfg.D)
    st = h.stats()
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("force64", [False, True])
def test_random_scenes_circle(seed, force64, cuda_device):
    rng = np.random.default_rng(7000 + seed)
    N = int(rng.choice([4, 7, 16, 33, 64, 128, 200]))
    D = int(rng.integers(1, 9))
    T = int(rng.choice([1, 2, 3, 8, 20]))
    pts = synth.random_scene(8000 + seed, N, max_lines=4, max_noise=int(rng.choice([10, 300, 3000])))
    ref = oracle.detect(pts, N, D, T, AB, variant=1)
    h = _run(pts, N, D, T, AB, cuda_device, force_int64=force64)
    compare_all(h, ref, AB, D)
    st = h.stats()
    assert (st["tests"], st["votes"]) == (ref.tests, ref.votes)
    assert st["int_bits"] == (64 if force64 else 32)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("force64", [False, True])
def test_random_scenes_circle_mb(seed, force64, cuda_device):
    rng = np.random.default_rng(9100 + seed)
    N = int(rng.choice([4, 7, 16, 33, 64, 128]))
    D = int(rng.integers(1, 8))
    T = int(rng.choice([2, 8, 20, 60]))
    pts = synth.random_scene(9200 + seed, N, max_lines=4, max_noise=int(rng.choice([10, 100, 600])))
    ref = oracle.detect(pts, N, D, T, AB, variant=2)
    h = _run(pts, N, D, T, AB, cuda_device, hht.FHT_CIRCLE_MB, force_int64=force64)
    compare_all(h, ref, AB, D)
    st = h.stats()
    assert (st["tests"], st["votes"]) == (ref.tests, ref.votes)
    assert st["int_bits"] == (64 if force64 else 32)


def test_circle_ranges_under_tiny_budget(cuda_device):
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves, variant=1)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, cuda_device, hht.FHT_CIRCLE, mem_budget=256 << 10)
    compare_all(h, ref, cfg.halves, cfg.D)
    assert h.stats()["ranges"] > 4 * cfg.D


def test_circle_mb_ranges_under_tiny_budget(cuda_device):
    N, D, T = 128, 7, 40
    pts = synth.random_scene(4242, N, max_lines=6, max_noise=800)
    ref = oracle.detect(pts, N, D, T, AB, variant=2)
    h = _run(pts, N, D, T, AB, cuda_device, hht.FHT_CIRCLE_MB, mem_budget=64 << 10)
    compare_all(h, ref, AB, D)
    assert h.stats()["ranges"] > 2 * D


@pytest.mark.parametrize("var", VARS)
@pytest.mark.parametrize("case", ["empty", "identical", "d1", "d2", "d3", "n1"])
def test_circle_edge_cases(case, var, cuda_device):
    N, D, T = 16, 4, 2
    if case == "empty":
        pts = np.zeros((0, 2), np.int32)
    elif case == "identical":
        pts, T = np.array([[5, 9]] * 300, np.int32), 100
    elif case == "n1":
        pts, N, D, T = np.array([[0, 0]] * 5, np.int32), 1, 3, 1
    else:
        D = int(case[1])
        pts = synth.random_scene(30 + D, 16, max_noise=60)
    ref = oracle.detect(pts, N, D, T, AB, variant=var)
    h = _run(pts, N, D, T, AB, cuda_device, var)
    compare_all(h, ref, AB, D)


@pytest.mark.parametrize("cid,var", CFG_VARS)
def test_circle_casts_extra_votes(cid, var, cuda_device):
    """North star: the circumcircle test (FHT) votes wherever the exact test does and more: at every
    region visited by both runs, votes_circle >= votes_exact; strictly more votes in total."""
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    he = hht.HHT(halves=cfg.halves)
    he.detect(_dev(pts, cuda_device), cfg.N, cfg.D, cfg.T)
    hc = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, cuda_device, var)
    for half in (1, 2):
        if not cfg.halves & half:
            continue
        for lev in range(cfg.D + 1):
            e = {(a, c): v for a, c, v in he.level(0, half, lev).tolist()}
            c = {(a, c): v for a, c, v in hc.level(0, half, lev).tolist()}
            assert set(e) <= set(c), f"level {lev}: exact visits a region the circle run does not"
            assert all(c[k] >= v for k, v in e.items()), f"level {lev}: circle votes < exact votes"
    assert hc.stats()["votes"] > he.stats()["votes"]


def test_circle_overflow_rejected(cuda_device):
    h = hht.HHT(halves=AB, variant=hht.FHT_CIRCLE)
    with pytest.raises(hht.HHTError) as e:
        h.detect(_dev(np.array([[0, 0]], np.int32), cuda_device), 65536, 30, 2)
    assert e.value.name == "HHT_EOVERFLOW"


def test_circle_mb_extremes(cuda_device):
    """Variant 2 compares in 128 bits: (1 + ex^2)(4 + 9N^2) s^2 < 2^125.2 for every tested region
    (children of the root down) within the API's limits (N <= 65536, depth <= 30), so it never
    overflows; at the extreme it runs and matches the oracle (ex = 0 keeps the oracle's own root
    test inside its signed 128-bit range)."""
    pts = np.array([[0, 0], [0, 65535], [0, 1]], np.int32)     # ALPHA lines b = 0, 65535, 1
    ref = oracle.detect(pts, 65536, 30, 2, hht.ALPHA, variant=2)
    h = _run(pts, 65536, 30, 2, hht.ALPHA, cuda_device, hht.FHT_CIRCLE_MB)
    assert ref.levels[(1, 1)].shape[0] == 4 and ref.levels[(1, 2)].shape[0] == 0
    for lev in range(3):
        assert np.array_equal(h.level(0, 1, lev), ref.levels[(1, lev)])
