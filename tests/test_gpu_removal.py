"""GPU solution() with point removal (hht_result_lines)
against the oracle's literal depth-first detector with removal on (oracle_detect_removal, pinned in
tests/test_oracle_removal.py): the emitted lines and their live votes must be identical, in order,
and so must each line's support (the points it removed). Config 3 in full against an oracle-written
digest (scripts/write_golden_removal.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


def _dev(pts, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(pts, dtype=np.int32)).to(dev)


def _check(h, pts, N, D, T, halves, image=0):
    lines, sup = oracle.detect_removal(pts, N, D, T, halves)
    got = h.lines(image)
    assert np.array_equal(got[:, 1:], lines.astype(np.int64)), (got[:5], lines[:5])
    assert (got[:, 0] == image).all()
    want = sup.astype(np.int64)
    want = want[np.lexsort((want[:, 1], want[:, 0]))] if want.shape[0] else want.reshape(0, 2)
    gs = h.line_points(image)
    assert np.array_equal(gs, want), (gs[:5], want[:5])


@pytest.mark.parametrize("cid", [1, 2])
def test_removal_configs(cid, cuda_device):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    h = hht.HHT(halves=cfg.halves)
    h.detect(_dev(pts, cuda_device), cfg.N, cfg.D, cfg.T)
    _check(h, pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    assert 0 < h.lines().shape[0] < h.leaves().shape[0]


@pytest.mark.parametrize("seed", range(16))
def test_removal_random(seed, cuda_device):
    rng = np.random.default_rng(1300 + seed)
    N = int(rng.choice([8, 16, 33, 64, 128]))
    D = int(rng.integers(1, 8))
    T = int(rng.choice([1, 2, 4, 9]))
    pts = synth.random_scene(1400 + seed, N, max_lines=4, max_noise=int(rng.choice([20, 200, 1000])))
    h = hht.HHT(halves=AB, force_int64=bool(seed % 2))
    h.detect(_dev(pts, cuda_device), N, D, T)
    _check(h, pts, N, D, T, AB)


def test_removal_batch_and_trees(cuda_device):
    N, D, T = 64, 6, 5
    imgs = [synth.random_scene(1500 + k, N, max_lines=3, max_noise=k * 60) for k in range(4)]
    imgs[2] = imgs[2][:0]
    offs = np.zeros(len(imgs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in imgs])
    h = hht.HHT(halves=AB)
    h.detect_batch(_dev(np.concatenate(imgs), cuda_device), offs, N, D, T)
    for b, p in enumerate(imgs):
        _check(h, p, N, D, T, AB, image=b)
    # per-tree point sets (edge front end layout): ALPHA and BETA trees on different points
    a = synth.random_scene(1600, N, max_lines=3, max_noise=100)
    bta = synth.random_scene(1601, N, max_lines=3, max_noise=100)
    h.detect_trees(np.concatenate([a, bta]).astype(np.int32), [0, len(a), len(a) + len(bta)], N, D, T)
    la, _ = oracle.detect_removal(a, N, D, T, hht.ALPHA)
    lb, _ = oracle.detect_removal(bta, N, D, T, hht.BETA)
    assert np.array_equal(h.lines()[:, 1:], np.concatenate([la, lb]).astype(np.int64))


def test_removal_rejects_circle(cuda_device):
    h = hht.HHT(halves=AB, variant=hht.FHT_CIRCLE)
    h.detect(_dev(synth.random_scene(5, 32, max_noise=50), cuda_device), 32, 5, 3)
    with pytest.raises(hht.HHTError) as e:
        h.lines()
    assert e.value.name == "HHT_EINVAL"


def test_removal_c3_digest(cuda_device):
    """Config 3 in full (400k points, 4.2e6 candidate leaves): lines and supports against the digest
    of oracle_detect_removal (tests/golden/c3_removal_digest.json)."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c3_removal_digest.json")))
    cfg = synth.CONFIGS[3]
    pts, _ = synth.config_image(3)
    h = hht.HHT(halves=cfg.halves)
    h.detect(_dev(pts, cuda_device), cfg.N, cfg.D, cfg.T)
    lines = h.lines()
    L = np.ascontiguousarray(lines[:, 1:].astype("<u4"))
    assert L.shape[0] == gold["lines"]
    assert hashlib.sha256(L.tobytes()).hexdigest() == gold["lines_sha256"]
    S = np.ascontiguousarray(h.line_points().astype("<u4"))
    assert S.shape[0] == gold["support"]
    assert hashlib.sha256(S.tobytes()).hexdigest() == gold["support_sha256"]
