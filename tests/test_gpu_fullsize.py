"""Full-size parity for BASELINE configs 3-5 in the launch configuration bench.py times.

The oracle's full outputs are too large to store, so scripts/write_golden.py (oracle only) wrote
sha256 digests of every (half, level) record array and of the leaf list; the GPU output must hash
identically (bit-exact). Independently of the digests, sampled regions are re-counted by brute
force over all points (oracle.region_votes) and the full output is checked for the tree invariants
(root = E, visited = children of split regions in quad order, child <= parent,
parent <= sum(children) <= 3*parent, tests recomputed from the records)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import check_structure

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _digest_check(h, cfg, images, gold):
    halves = [x for x in (1, 2) if cfg.halves & x]
    for half in halves:
        for lev in range(cfg.D + 1):
            arrs = [h.level(b, half, lev) for b in range(images)]
            arr = np.ascontiguousarray(np.concatenate(arrs).astype("<u4"))
            key = f"{half}/{lev}"
            assert arr.shape[0] == gold["level_count"][key], (key, arr.shape[0], gold["level_count"][key])
            assert hashlib.sha256(arr.tobytes()).hexdigest() == gold["level_sha256"][key], key
    lv = np.ascontiguousarray(h.leaves(-1).astype("<u4"))
    assert lv.shape[0] == gold["leaves"]
    assert hashlib.sha256(lv.tobytes()).hexdigest() == gold["leaves_sha256"]
    st = h.stats()
    assert st["tests"] == gold["tests"] and st["votes"] == gold["votes"]


def _sampled_brute(h, pts, cfg, image, nsamp, rng):
    """Re-count sampled visited regions over ALL points; sampled leaf cells: emitted iff votes > T."""
    for half in [x for x in (1, 2) if cfg.halves & x]:
        for lev in range(cfg.D + 1):
            recs = h.level(image, half, lev)
            if recs.shape[0] == 0:
                continue
            for k in rng.choice(recs.shape[0], size=min(nsamp, recs.shape[0]), replace=False):
                a, c, v = (int(x) for x in recs[k])
                assert oracle.region_votes(pts, half, cfg.N, cfg.D, lev, a, c) == v, (half, lev, a, c)
        leaves = h.leaves(image)
        cells = {(int(i), int(j)) for _, hh, i, j, _ in leaves.tolist() if hh == half}
        side = 1 << cfg.D
        for _ in range(nsamp):
            i, j = int(rng.integers(side)), int(rng.integers(side))
            v = oracle.region_votes(pts, half, cfg.N, cfg.D, cfg.D, i, j)
            assert ((i, j) in cells) == (v > cfg.T), (half, i, j, v)


@pytest.mark.parametrize("cid,int64", [(3, False), (4, False), (5, False), (3, True), (4, True), (5, True)])
def test_fullsize_config(cid, int64, cuda_device):
    """The bench's launch configuration (int32, where exact for every config), and the int64
    instantiation north_star names on configs 3-5, against the oracle's digests."""
    import torch
    path = os.path.join(GOLD, f"c{cid}_digest.json")
    cfg = synth.CONFIGS[cid]
    if cfg.images > 1:
        pts, offs = synth.config_batch(cid)
    else:
        pts, _ = synth.config_image(cid)
        offs = np.array([0, pts.shape[0]])
    h = hht.HHT(halves=cfg.halves, profile=True, force_int64=int64)   # profile on: as bench.py runs
    h.detect_batch(torch.from_numpy(pts).to(cuda_device), offs, cfg.N, cfg.D, cfg.T)
    assert h.stats()["int_bits"] == (64 if int64 else 32)
    images = offs.shape[0] - 1
    assert os.path.exists(path), f"missing oracle digest {path} (scripts/write_golden.py --config {cid})"
    _digest_check(h, cfg, images, json.load(open(path)))
    if int64:
        return
    # structure of every tree (full output), sampled brute-force counts on image 0
    tests = 0
    for b in range(images if images <= 4 else 4):
        for half in [x for x in (1, 2) if cfg.halves & x]:
            levels = [h.level(b, half, l) for l in range(cfg.D + 1)]
            t, _ = check_structure(levels, int(offs[b + 1] - offs[b]), cfg.T, cfg.D)
            tests += t
    if images == 1:
        assert tests == h.stats()["tests"]
    rng = np.random.default_rng(cid)
    p0 = pts[offs[0]:offs[1]]
    _sampled_brute(h, p0, cfg, 0, 3 if cid == 5 else 30, rng)


@pytest.mark.parametrize("cid", [3, 5])
def test_fullsize_e2e_leaf_sink(cid, cuda_device):
    """bench.py's e2e configuration (profile on, pinned HOST points staged by the library, the
    detected lines streamed to a pinned host sink during the call, default memory budget): the
    streamed (image, half, i, j, votes) rows hash to the oracle digest's leaves, in order."""
    import torch
    cfg = synth.CONFIGS[cid]
    gold = json.load(open(os.path.join(GOLD, f"c{cid}_digest.json")))
    pts, _ = synth.config_image(cid)
    offs = np.array([0, pts.shape[0]], dtype=np.int64)
    host = torch.from_numpy(np.ascontiguousarray(pts)).pin_memory().numpy()
    h = hht.HHT(halves=cfg.halves, profile=True)
    sink = torch.empty((gold["leaves"] + 1024, 5), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    h.set_leaf_sink(sink)
    h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)
    st = h.stats()
    assert st["leaves_streamed"] == st["leaves"] == gold["leaves"]
    rows = np.ascontiguousarray(sink[:gold["leaves"]].astype("<u4"))
    assert hashlib.sha256(rows.tobytes()).hexdigest() == gold["leaves_sha256"]
    assert st["tests"] == gold["tests"] and st["votes"] == gold["votes"]
    h.close()


@pytest.mark.parametrize("cid", [3, 5])
def test_fullsize_e2e_leaf_sink_packed(cid, cuda_device):
    """bench.py's e2e configuration with the packed sink (8-byte rows + per-tree offsets): the rows,
    expanded to (image, half, i, j, votes), hash to the oracle digest's leaves, in order."""
    import torch
    from tests.test_gpu_parity import _unpack_rows
    cfg = synth.CONFIGS[cid]
    gold = json.load(open(os.path.join(GOLD, f"c{cid}_digest.json")))
    pts, _ = synth.config_image(cid)
    offs = np.array([0, pts.shape[0]], dtype=np.int64)
    host = torch.from_numpy(np.ascontiguousarray(pts)).pin_memory().numpy()
    h = hht.HHT(halves=cfg.halves, profile=True)
    sink = torch.empty(gold["leaves"] + 1024, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    h.set_leaf_sink_packed(sink)
    h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)
    st = h.stats()
    assert st["leaves_streamed"] == st["leaves"] == gold["leaves"]
    rows = _unpack_rows(sink[:gold["leaves"]], h.tree_offsets(), 2, cfg.halves)
    rows = np.ascontiguousarray(rows.astype("<u4"))
    assert hashlib.sha256(rows.tobytes()).hexdigest() == gold["leaves_sha256"]
    assert st["tests"] == gold["tests"] and st["votes"] == gold["votes"]
    h.close()
