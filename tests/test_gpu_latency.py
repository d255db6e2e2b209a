"""The one-launch latency path (k_small; opts.latency_path): tiny detections run every level inside
one 1024-thread block. Its records, leaves and statistics must equal the oracle's and the
multi-kernel path's, bit for bit."""
import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import compare_all

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


def eligible(n_per_tree, D, T):
    """Mirror of the library's admission rule (hht_driver.cu small_bounds / small_mode): 1 = k_small
    (everything in shared memory when it fits 220 KiB; else lists in device memory up to 2^16 entries
    with the frontier arrays in shared memory); 2 = k_mid (one cooperative launch, lists up to 2^26
    entries per level); 0 = the multi-kernel path."""
    S = max(sum(n_per_tree) * ((1 << D) - 1), 1)
    F = min(S // (T + 1) + len(n_per_tree) + 1, S + 1)
    if (4 * (2 * S + 8 * (F + 1) + 8 * F) <= 220 * 1024
            or (S <= (1 << 16) and 4 * (8 * (F + 1) + 8 * F) <= 220 * 1024)):
        return 1
    return 2 if (S <= (1 << 26) and F + 1 <= 3072 * 256 and D <= 24) else 0


def _dev(pts, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(pts, dtype=np.int32)).to(dev)


@pytest.mark.parametrize("seed", range(40))
def test_latency_path_random(seed, cuda_device):
    rng = np.random.default_rng(2100 + seed)
    N = int(rng.choice([4, 7, 16, 33, 64, 128, 256]))
    D = int(rng.integers(1, 7))
    T = int(rng.choice([1, 2, 3, 8, 20]))
    halves = [AB, hht.ALPHA, hht.BETA][seed % 3]
    pts = synth.random_scene(2200 + seed, N, max_lines=4, max_noise=int(rng.choice([10, 100, 400])))
    ref = oracle.detect(pts, N, D, T, halves)
    h = hht.HHT(halves=halves, force_int64=bool(seed % 4 == 0))
    h.detect(_dev(pts, cuda_device), N, D, T)
    st = h.stats()
    ntrees = bin(halves).count("1")
    assert st["latency_path"] == eligible([len(pts)] * ntrees, D, T)
    compare_all(h, ref, halves, D)
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])
    hm = hht.HHT(halves=halves, latency_path=2)
    hm.detect(_dev(pts, cuda_device), N, D, T)
    sm = hm.stats()
    assert sm["latency_path"] == 0
    assert (sm["visited"], sm["split"]) == (st["visited"], st["split"])


@pytest.mark.parametrize("cid", [1])
def test_latency_path_config(cid, cuda_device):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    h = hht.HHT(halves=cfg.halves)
    h.detect(_dev(pts, cuda_device), cfg.N, cfg.D, cfg.T)
    assert h.stats()["latency_path"] == 1
    compare_all(h, oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves), cfg.halves, cfg.D)


@pytest.mark.parametrize("case", ["empty", "below_threshold", "identical", "d1", "n1", "batch"])
def test_latency_path_edges(case, cuda_device):
    N, D, T = 16, 4, 2
    if case == "batch":
        imgs = [synth.random_scene(2300 + k, 32, max_lines=3, max_noise=k * 30) for k in range(5)]
        imgs[1] = imgs[1][:0]
        offs = np.zeros(6, dtype=np.int64)
        offs[1:] = np.cumsum([len(p) for p in imgs])
        h = hht.HHT(halves=AB)
        sink = np.zeros((4096, 5), np.uint32)
        h.set_leaf_sink(sink)
        h.detect_batch(_dev(np.concatenate(imgs), cuda_device), offs, 32, 5, 3)
        assert h.stats()["latency_path"] == 1
        for b, p in enumerate(imgs):
            compare_all(h, oracle.detect(p, 32, 5, 3, AB), AB, 5, image=b)
        n = h.stats()["leaves_streamed"]
        assert n == h.stats()["leaves"] and np.array_equal(sink[:n].astype(np.int64), h.leaves(-1))
        return
    if case == "empty":
        pts = np.zeros((0, 2), np.int32)
    elif case == "below_threshold":
        pts = np.array([[1, 2], [3, 4]], np.int32)
    elif case == "identical":
        pts, T = np.array([[5, 9]] * 300, np.int32), 100
    elif case == "d1":
        pts, D = synth.random_scene(3, 16, max_noise=40), 1
    else:
        pts, N, D, T = np.array([[0, 0]] * 5, np.int32), 1, 3, 1
    h = hht.HHT(halves=AB)
    h.detect(_dev(pts, cuda_device), N, D, T)
    compare_all(h, oracle.detect(pts, N, D, T, AB), AB, D)


@pytest.mark.parametrize("size,seed", [(48, 2), (48, 3), (48, 4), (64, 3), (64, 5), (64, 7)])
def test_latency_path_device_scratch(size, seed, cuda_device):
    """Scenes whose lists exceed shared memory but stay under 2^16 entries run the one-launch path
    with the lists in device memory (frontier arrays in shared memory); identical to the oracle."""
    D, T = 6, 8
    pts = synth.random_scene(2400 + 10 * size + seed, size, max_lines=5, max_noise=size * 3)
    n = [len(pts), len(pts)]
    S = sum(n) * ((1 << D) - 1)
    F = min(S // (T + 1) + 3, S + 1)
    assert 4 * (2 * S + 8 * (F + 1) + 8 * F) > 220 * 1024 and eligible(n, D, T)   # the device-list mode
    ref = oracle.detect(pts, size, D, T, AB)
    h = hht.HHT(halves=AB)
    h.detect(_dev(pts, cuda_device), size, D, T)
    st = h.stats()
    assert st["latency_path"] == 1, S
    compare_all(h, ref, AB, D)
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])


@pytest.mark.parametrize("seed", range(30))
def test_mid_path_random(seed, cuda_device):
    """k_mid (opts.latency_path = 3 forces it): records, leaves and statistics bit-exact against the
    oracle, and visited/split counts equal to the multi-kernel path's."""
    rng = np.random.default_rng(3100 + seed)
    N = int(rng.choice([4, 16, 33, 64, 128, 256, 512]))
    D = int(rng.integers(1, 10))
    T = int(rng.choice([1, 2, 5, 20, 60]))
    halves = [AB, hht.ALPHA, hht.BETA][seed % 3]
    pts = synth.random_scene(3200 + seed, N, max_lines=5, max_noise=int(rng.choice([10, 300, 3000])))
    ref = oracle.detect(pts, N, D, T, halves)
    h = hht.HHT(halves=halves, latency_path=3, force_int64=bool(seed % 4 == 1))
    h.detect(_dev(pts, cuda_device), N, D, T)
    st = h.stats()
    assert st["latency_path"] == 2
    compare_all(h, ref, halves, D)
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])
    hm = hht.HHT(halves=halves, latency_path=2)
    hm.detect(_dev(pts, cuda_device), N, D, T)
    sm = hm.stats()
    assert (sm["visited"], sm["split"]) == (st["visited"], st["split"])


def test_mid_path_config2_and_batch(cuda_device):
    """Config 2 runs on k_mid by default (bounds admit it) and equals the oracle in full; a ragged
    batch with an empty image too."""
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    h = hht.HHT(halves=cfg.halves)
    h.detect(_dev(pts, cuda_device), cfg.N, cfg.D, cfg.T)
    assert h.stats()["latency_path"] == 2
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    compare_all(h, ref, cfg.halves, cfg.D)
    st = h.stats()
    assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])
    imgs = [synth.random_scene(3300 + k, 128, max_lines=3, max_noise=k * 400) for k in range(4)]
    imgs[1] = imgs[1][:0]
    offs = np.zeros(5, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in imgs])
    hb = hht.HHT(halves=AB, latency_path=3)
    hb.detect_batch(_dev(np.concatenate(imgs), cuda_device), offs, 128, 7, 6)
    assert hb.stats()["latency_path"] == 2
    for b, p in enumerate(imgs):
        compare_all(hb, oracle.detect(p, 128, 7, 6, AB), AB, 7, image=b)


def test_mid_path_range_error(cuda_device):
    h = hht.HHT(halves=AB, latency_path=3)
    with pytest.raises(hht.HHTError) as e:
        h.detect(_dev(np.array([[0, 0], [70, 1]], np.int32), cuda_device), 64, 6, 1)
    assert e.value.name == "HHT_ERANGE"


@pytest.mark.gpu
def test_small_path_range_error_then_recovers(cuda_device):
    """k_small stages and range-checks the points itself: an out-of-range point fails the call with
    HHT_ERANGE on the one-block path, and the next call on the same context is exact."""
    h = hht.HHT(halves=AB)
    with pytest.raises(hht.HHTError) as e:
        h.detect(_dev(np.array([[0, 0], [3, 64]], np.int32), cuda_device), 64, 6, 1)
    assert e.value.name == "HHT_ERANGE"
    pts = synth.random_scene(4100, 64, max_lines=3, max_noise=40)
    h.detect(_dev(pts, cuda_device), 64, 6, 4)
    assert h.stats()["latency_path"] == 1
    compare_all(h, oracle.detect(pts, 64, 6, 4, AB), AB, 6)


@pytest.mark.gpu
def test_small_path_constant_blocks_across_shapes(cuda_device):
    """The latency path skips re-uploading its constant blocks (tree offsets, record pointers, half
    flags) when a call repeats the previous one's; alternating shapes, halves and batch sizes on one
    context must still match the oracle every time."""
    h = hht.HHT(halves=AB)
    ha = hht.HHT(halves=hht.ALPHA)
    scenes = [(synth.random_scene(4200 + k, N, max_lines=3, max_noise=30), N, D, T)
              for k, (N, D, T) in enumerate([(64, 6, 4), (32, 5, 3), (64, 6, 4), (128, 7, 6), (32, 5, 3)])]
    for rep in range(2):
        for pts, N, D, T in scenes:
            for ctx, halves in ((h, AB), (ha, hht.ALPHA)):
                ctx.detect(_dev(pts, cuda_device), N, D, T)
                assert ctx.stats()["latency_path"] in (1, 2)   # k_small, or k_mid (128 px: its block overwrites)
                compare_all(ctx, oracle.detect(pts, N, D, T, halves), halves, D)
    imgs = [synth.random_scene(4300 + k, 64, max_lines=2, max_noise=20) for k in range(3)]
    for nb in (3, 2, 3):
        offs = np.zeros(nb + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(p) for p in imgs[:nb]])
        h.detect_batch(_dev(np.concatenate(imgs[:nb]), cuda_device), offs, 64, 6, 4)
        assert h.stats()["latency_path"] == 1
        for b in range(nb):
            compare_all(h, oracle.detect(imgs[b], 64, 6, 4, AB), AB, 6, image=b)
