"""GPU parity: libhht (CUDA, through the C ABI) vs the CPU oracle, element by element.

Records of every level (a, c, votes), the leaf list, and the tests/votes statistics must be
identical (integer work: bit-exact). Sizes span many 256-entry chunks and ragged
tails; edge cases cover empty input, E <= T, identical points, D = 1/2, the int64 kernels,
depth-first list ranges under a tiny memory budget, host-pointer input, batches with empty images,
and the error paths."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import check_structure, compare_all

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


@pytest.fixture(scope="module")
def torch_dev(cuda_device):
    return cuda_device


def _dev(pts, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(pts, dtype=np.int32)).to(dev)


def _run(pts, N, D, T, halves, dev, **kw):
    kw.setdefault("latency_path", 2)      # the multi-kernel path; the one-launch path: test_gpu_latency.py
    h = hht.HHT(halves=halves, **kw)
    h.detect(_dev(pts, dev), N, D, T)
    return h


def test_survey_example(torch_dev):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_example_n8_d3_t2.json")))
    pts = np.array(g["points"], dtype=np.int32)
    h = _run(pts, 8, 3, 2, hht.ALPHA, torch_dev)
    for lev, recs in g["levels"].items():
        assert h.level(0, hht.ALPHA, int(lev)).tolist() == recs
    assert h.leaves(0)[:, 2:].tolist() == g["leaves"]
    st = h.stats()
    assert st["votes"] == g["votes"] and st["tests"] == g["tests"]


@pytest.mark.parametrize("cid", [1, 2])
def test_config_full_parity(cid, torch_dev):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, torch_dev)
    compare_all(h, ref, cfg.halves, cfg.D)
    st = h.stats()
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])
    assert st["int_bits"] == 32


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("force64", [False, True])
def test_random_scenes(seed, force64, torch_dev):
    rng = np.random.default_rng(seed)
    N = int(rng.choice([4, 7, 16, 33, 64, 128, 200]))
    D = int(rng.integers(1, 9))
    T = int(rng.choice([1, 2, 3, 8, 20]))
    pts = synth.random_scene(1000 + seed, N, max_lines=4, max_noise=int(rng.choice([10, 300, 3000])))
    ref = oracle.detect(pts, N, D, T, AB)
    h = _run(pts, N, D, T, AB, torch_dev, force_int64=force64)
    compare_all(h, ref, AB, D)
    st = h.stats()
    assert (st["tests"], st["votes"]) == (ref.tests, ref.votes)
    assert st["int_bits"] == (64 if force64 else 32)


def test_depth_beyond_log2n_int64(torch_dev):
    """D > log2 N and 5*N*2^D > 2^31: the library switches to the int64 kernels by itself."""
    pts = synth.random_scene(77, 100, max_lines=2, max_noise=50)
    N, D, T = 100, 23, 10
    ref = oracle.detect(pts, N, D, T, AB)
    h = _run(pts, N, D, T, AB, torch_dev)
    assert h.stats()["int_bits"] == 64
    compare_all(h, ref, AB, D)


def test_ranges_under_tiny_budget(torch_dev):
    """A 256 KiB list budget forces many depth-first ranges; output must not change."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, torch_dev, mem_budget=256 << 10)
    compare_all(h, ref, cfg.halves, cfg.D)
    assert h.stats()["ranges"] > 4 * cfg.D


def test_host_pointer_input(torch_dev):
    cfg = synth.CONFIGS[1]
    pts, _ = synth.config_image(1)
    h = hht.HHT(halves=cfg.halves)
    h.detect(pts, cfg.N, cfg.D, cfg.T)          # numpy (host) pointer: staged by the library
    st = h.stats()
    assert st["h2d_bytes"] == pts.nbytes
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    compare_all(h, ref, cfg.halves, cfg.D)


def test_batch_with_empty_and_ragged_images(torch_dev):
    N, D, T = 64, 6, 6
    imgs = [synth.random_scene(500 + k, N, max_lines=3, max_noise=k * 40) for k in range(6)]
    imgs[2] = np.zeros((0, 2), dtype=np.int32)
    imgs[4] = imgs[4][:3]
    offs = np.zeros(len(imgs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in imgs])
    allp = np.concatenate(imgs).astype(np.int32)
    h = hht.HHT(halves=AB)
    h.detect_batch(_dev(allp, torch_dev), offs, N, D, T)
    tests = votes = 0
    for b, p in enumerate(imgs):
        ref = oracle.detect(p, N, D, T, AB)
        compare_all(h, ref, AB, D, image=b)
        tests += ref.tests
        votes += ref.votes
    st = h.stats()
    assert (st["tests"], st["votes"]) == (tests, votes)
    allv = h.leaves(-1)
    assert (np.diff(allv[:, 0]) >= 0).all()


@pytest.mark.parametrize("case", ["empty", "below_threshold", "identical", "d1", "d2", "n1", "corner_touch"])
def test_edge_cases(case, torch_dev):
    N, D, T, halves = 16, 4, 2, AB
    if case == "empty":
        pts = np.zeros((0, 2), np.int32)
    elif case == "below_threshold":
        pts = np.array([[1, 2], [3, 4]], np.int32)
    elif case == "identical":
        pts = np.array([[5, 9]] * 300, np.int32)
        T = 100
    elif case == "d1":
        pts = synth.random_scene(3, 16, max_noise=40)
        D = 1
    elif case == "d2":
        pts = synth.random_scene(4, 16, max_noise=40)
        D = 2
    elif case == "n1":
        pts = np.array([[0, 0]] * 5, np.int32)
        N, D, T = 1, 3, 1
    else:   # an NE-corner touch from below votes, an SW touch does not
        pts = np.array([[4, 4]] * 3, np.int32)
        N, D, T, halves = 8, 3, 1, hht.ALPHA
    ref = oracle.detect(pts, N, D, T, halves)
    h = _run(pts, N, D, T, halves, torch_dev)
    compare_all(h, ref, halves, D)
    if case == "corner_touch":
        cells = {(int(i), int(j)) for _, _, i, j, _ in h.leaves(0).tolist()}
        assert (3, 3) in cells and (4, 4) not in cells


def test_errors(torch_dev):
    h = hht.HHT(halves=AB)
    bad = np.array([[0, 0], [16, 3]], np.int32)
    with pytest.raises(hht.HHTError) as e:
        h.detect(_dev(bad, torch_dev), 16, 4, 2)
    assert e.value.name == "HHT_ERANGE"
    ok = np.array([[0, 0]], np.int32)
    for N, D, T in [(0, 4, 2), (16, 0, 2), (16, 4, 0), (70000, 4, 2), (16, 31, 2)]:
        with pytest.raises(hht.HHTError) as e:
            h.detect(_dev(ok, torch_dev), N, D, T)
        assert e.value.name == "HHT_EINVAL"
    with pytest.raises(hht.HHTError) as e:
        h.level(0, hht.ALPHA, 0)          # no successful detect since the errors
    assert e.value.name == "HHT_ESTATE"


def test_records_off_still_emits_leaves(torch_dev):
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, torch_dev, record_levels=False)
    assert np.array_equal(h.leaves(0)[:, 1:], ref.leaves.astype(np.int64))
    with pytest.raises(hht.HHTError):
        h.level(0, hht.ALPHA, 1)


def test_repeat_calls_identical(torch_dev):
    """Determinism across calls on one context (outputs are order-independent counts)."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    h = hht.HHT(halves=cfg.halves)
    d = _dev(pts, torch_dev)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    a = [h.level(0, 2, l).copy() for l in range(cfg.D + 1)], h.leaves().copy()
    h.detect(d, cfg.N, cfg.D, cfg.T)
    b = [h.level(0, 2, l) for l in range(cfg.D + 1)], h.leaves()
    assert all(np.array_equal(x, y) for x, y in zip(a[0], b[0])) and np.array_equal(a[1], b[1])


def test_c2_structure_and_profile(torch_dev):
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    h = _run(pts, cfg.N, cfg.D, cfg.T, cfg.halves, torch_dev, profile=True)
    for half in (1, 2):
        levels = [h.level(0, half, l) for l in range(cfg.D + 1)]
        check_structure(levels, pts.shape[0], cfg.T, cfg.D)
    prof = h.profile()
    assert prof["write"]["launches"] > 0 and prof["split"]["launches"] >= cfg.D


@pytest.mark.parametrize("tail_depth", [3, 4, 5, 6])
@pytest.mark.parametrize("seed", range(8))
def test_tail_depth_variants(seed, tail_depth, torch_dev):
    """The 8x8 (D-3), 16x16 (D-4), fused 16x16-from-(D-5) and fused 16x16-from-(D-6) tails give
    identical records and leaves."""
    rng = np.random.default_rng(100 + seed)
    N = int(rng.choice([16, 33, 64, 200]))
    D = int(rng.integers(3, 9))
    T = int(rng.choice([1, 2, 5, 12]))
    pts = synth.random_scene(3000 + seed, N, max_lines=4, max_noise=int(rng.choice([50, 500, 4000])))
    ref = oracle.detect(pts, N, D, T, AB)
    h = _run(pts, N, D, T, AB, torch_dev, tail_depth=tail_depth)
    compare_all(h, ref, AB, D)
    assert (h.stats()["tests"], h.stats()["votes"]) == (ref.tests, ref.votes)


@pytest.mark.parametrize("prefetch", [1, 2, 3])
@pytest.mark.parametrize("seed", range(6))
def test_prefetch_modes(seed, prefetch, torch_dev):
    """The list passes' work loop with the descriptor prefetched only (1), with the next chunk's
    entries in registers (2), and with a bulk-copy (cp.async.bulk + mbarrier) ring two chunks ahead
    (3) give identical results, including many ranges (list bases) and int64."""
    rng = np.random.default_rng(800 + seed)
    N = int(rng.choice([64, 200, 256]))
    D = int(rng.integers(6, 10))
    T = int(rng.choice([1, 3, 8]))
    pts = synth.random_scene(8100 + seed, N, max_lines=5, max_noise=int(rng.choice([500, 4000])))
    ref = oracle.detect(pts, N, D, T, AB)
    for budget in (0, 128 << 10):
        h = _run(pts, N, D, T, AB, torch_dev, prefetch=prefetch, mem_budget=budget, force_int64=bool(seed % 2))
        compare_all(h, ref, AB, D)
        assert (h.stats()["tests"], h.stats()["votes"]) == (ref.tests, ref.votes)


@pytest.mark.parametrize("tail_units", [0, 2, 3])
@pytest.mark.parametrize("seed", range(6))
def test_fused_tail_work_units(seed, tail_units, torch_dev):
    """The fused tail with each parent's chunks split into work units (auto: fewer parents than
    8 x warps), with one unit per parent (tail_units 2) and with whole parents followed by the last
    ones in 32-chunk pieces (tail_units 3, the many-parents scheme) give identical records and
    leaves, also under a small budget (many ranges, some with very few parents)."""
    rng = np.random.default_rng(700 + seed)
    N = int(rng.choice([64, 200, 256]))
    D = int(rng.integers(6, 9))
    T = int(rng.choice([1, 3, 8]))
    pts = synth.random_scene(7100 + seed, N, max_lines=5, max_noise=int(rng.choice([500, 4000])))
    ref = oracle.detect(pts, N, D, T, AB)
    for budget in (0, 128 << 10):
        h = _run(pts, N, D, T, AB, torch_dev, tail_units=tail_units, mem_budget=budget)
        compare_all(h, ref, AB, D)
        assert (h.stats()["tests"], h.stats()["votes"]) == (ref.tests, ref.votes)


def test_nccl_collectives_one_rank(torch_dev):
    """world = 1 with an NCCL id runs every collective call site (argument check, per-image
    counts, range agreement, per-level vote allreduce, error flag) on a 1-rank communicator;
    results must equal the oracle's."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    h = hht.HHT(halves=cfg.halves, nccl_id=hht.nccl_unique_id(), world=1, rank=0, mem_budget=1 << 20)
    h.detect(_dev(pts, torch_dev), cfg.N, cfg.D, cfg.T)
    compare_all(h, ref, cfg.halves, cfg.D)
    assert h.stats()["ranges"] > cfg.D
    imgs = [synth.random_scene(900 + k, 64, max_noise=200) for k in range(3)]
    offs = np.zeros(4, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in imgs])
    h.detect_batch(_dev(np.concatenate(imgs), torch_dev), offs, 64, 6, 5)
    for b, p in enumerate(imgs):
        compare_all(h, oracle.detect(p, 64, 6, 5, AB), AB, 6, image=b)
    bad = np.array([[0, 0], [70, 3]], np.int32)
    with pytest.raises(hht.HHTError) as e:
        h.detect(_dev(bad, torch_dev), 64, 6, 5)
    assert e.value.name == "HHT_ERANGE"


@pytest.mark.parametrize("budget", [0, 256 << 10])
def test_leaf_sink_streaming(budget, torch_dev):
    """hht_set_leaf_sink: rows streamed during the detect equal hht_result_leaves(-1) (same order),
    also across depth-first ranges; a too-small sink receives the first `cap` rows only."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    h = hht.HHT(halves=cfg.halves, mem_budget=budget)
    d = _dev(pts, torch_dev)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    want = h.leaves(-1)
    sink = np.zeros((want.shape[0] + 7, 5), dtype=np.uint32)
    h.set_leaf_sink(sink)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    st = h.stats()
    assert st["leaves_streamed"] == st["leaves"] == want.shape[0]
    assert np.array_equal(sink[:want.shape[0]].astype(np.int64), want)
    assert st["d2h_bytes"] >= 20 * want.shape[0]
    small = np.zeros((100, 5), dtype=np.uint32)
    h.set_leaf_sink(small)
    h.detect(pts, cfg.N, cfg.D, cfg.T)            # host input too
    st = h.stats()
    assert st["leaves_streamed"] == 100 and st["leaves"] == want.shape[0]
    assert np.array_equal(small.astype(np.int64), want[:100])
    h.set_leaf_sink(None)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    assert h.stats()["leaves_streamed"] == 0


def _unpack_rows(packed, offs, H, halves):
    """packed uint64 rows + per-tree offsets -> (image, half, i, j, votes) rows (hht_leaf order)."""
    hs = [x for x in (hht.ALPHA, hht.BETA) if halves & x]
    tree = np.repeat(np.arange(len(offs) - 1), np.diff(offs.astype(np.int64)))
    return np.stack([tree // H, np.array(hs, np.int64)[tree % H], (packed >> 48).astype(np.int64),
                     ((packed >> 32) & 0xFFFF).astype(np.int64), (packed & 0xFFFFFFFF).astype(np.int64)], axis=1)


@pytest.mark.parametrize("budget", [0, 256 << 10])
def test_leaf_sink_packed(budget, torch_dev):
    """hht_set_leaf_sink_packed: 8-byte rows (i << 48 | j << 32 | votes) streamed during the detect,
    with hht_result_tree_offsets, reproduce hht_result_leaves(-1) row for row, across depth-first
    ranges and for a ragged batch with empty images; 8 bytes per row over PCIe; depth > 16 refused."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    h = hht.HHT(halves=cfg.halves, mem_budget=budget)
    d = _dev(pts, torch_dev)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    want = h.leaves(-1)
    sink = np.zeros(want.shape[0] + 5, dtype=np.uint64)
    h.set_leaf_sink_packed(sink)
    h.detect(d, cfg.N, cfg.D, cfg.T)
    st = h.stats()
    assert st["leaves_streamed"] == st["leaves"] == want.shape[0]
    offs = h.tree_offsets()
    assert offs.shape[0] == 3 and offs[0] == 0 and offs[-1] == want.shape[0]
    assert np.array_equal(_unpack_rows(sink[:want.shape[0]], offs, 2, cfg.halves), want)
    assert st["d2h_bytes"] >= 8 * want.shape[0] and st["d2h_bytes"] < 20 * want.shape[0]
    # a ragged batch (empty images included), ALPHA only
    parts = [synth.random_scene(300 + k, 64, max_lines=3, max_noise=200) if k % 3 else np.zeros((0, 2), np.int32)
             for k in range(7)]
    allp = np.concatenate(parts).astype(np.int32)
    bo = np.concatenate([[0], np.cumsum([len(q) for q in parts])]).astype(np.int64)
    hb = hht.HHT(halves=hht.ALPHA, mem_budget=budget)
    hb.detect_batch(_dev(allp, torch_dev), bo, 64, 6, 4)
    want = hb.leaves(-1)
    sink = np.zeros(max(want.shape[0], 1), dtype=np.uint64)
    hb.set_leaf_sink_packed(sink)
    hb.detect_batch(_dev(allp, torch_dev), bo, 64, 6, 4)
    offs = hb.tree_offsets()
    assert offs.shape[0] == 8
    assert np.array_equal(_unpack_rows(sink[:want.shape[0]], offs, 1, hht.ALPHA), want)
    for b in range(7):
        assert offs[b + 1] - offs[b] == hb.leaves(b).shape[0]
    with pytest.raises(hht.HHTError) as e:
        hb.detect_batch(_dev(allp, torch_dev), bo, 64, 17, 4)
    assert e.value.name == "HHT_EINVAL"
    hb.set_leaf_sink_packed(None)
    hb.detect_batch(_dev(allp, torch_dev), bo, 64, 6, 4)
    assert hb.stats()["leaves_streamed"] == 0


@pytest.mark.parametrize("tail_depth", [4, 5, 6])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 1023, 4095, 16383, 32767])
def test_raster_fixed_point_extremes(N, tail_depth, torch_dev):
    """The 16x16 raster's fixed-point floors (csrc Raster16) at the extremes of 3N:
    smallest N (fx_s = 7) and the largest image sizes (2^24 / 3N down to 170), against the oracle."""
    D = 5 if N <= 5 else 8
    if N <= 5:                                   # tiny images: every pixel, several times
        xs, ys = np.meshgrid(np.arange(N), np.arange(N))
        pts = np.repeat(np.stack([xs.ravel(), ys.ravel()], 1).astype(np.int32), 7, axis=0)
    elif N < 16384:
        pts = synth.random_scene(500 + N, N, max_lines=4, max_noise=400)
    else:                                        # beyond the scene generator's range: noise + 2 lines
        rng = np.random.default_rng(N)
        i = np.arange(0, N, 37)
        pts = np.concatenate([rng.integers(0, N, (600, 2)), np.stack([i, (3 * i) // 5 + 11], 1),
                              np.stack([(2 * i) // 7 + 5, i], 1)]).astype(np.int32)
    T = 2
    ref = oracle.detect(pts, N, D, T, AB)
    h = _run(pts, N, D, T, AB, torch_dev, tail_depth=tail_depth)
    compare_all(h, ref, AB, D)
    assert (h.stats()["tests"], h.stats()["votes"]) == (ref.tests, ref.votes)
