"""The multi-rank path on one GPU: W contexts in one process, one host thread each, joined by an
in-process collective group (include/hht.h hht_group_create). Every collective the NCCL path makes
(argument agreement, per-image point counts, error flag, range agreement, per-level vote
allreduce, tail-grid allreduce) runs in the same order through a host-staged allreduce, so the
logic that differs between ranks — local candidate lists and list lengths against global votes,
agreed depth-first ranges — is checked bit-exactly against the oracle on the whole image. Points
are sharded contiguously as bench.py shards them (paper_1007_0547_b200/dist.py)."""
import threading

import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import compare_all

pytestmark = pytest.mark.gpu

AB = hht.ALPHA | hht.BETA


def _run_ranks(pts, N, D, T, halves, world, dev, setup=None, **kw):
    import torch
    g = hht.Group(world)
    hs = [hht.HHT(halves=halves, rank=r, world=world, group=g, **kw) for r in range(world)]
    if setup:
        for h in hs:
            setup(h)
    errs = [None] * world
    bounds = [synth.shard(pts.shape[0], r, world) for r in range(world)]
    shards = [torch.from_numpy(np.ascontiguousarray(pts[lo:hi])).to(dev) for lo, hi in bounds]

    def work(r):
        try:
            hs[r].detect(shards[r], N, D, T)
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return hs, g, errs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kw", [{}, {"tail_depth": 4}, {"tail_depth": 3}, {"tail_depth": 6},
                                {"mem_budget": 256 << 10}, {"mem_budget": 256 << 10, "tail_depth": 6},
                                {"variant": 1}])
def test_multirank_c2(world, kw, cuda_device):
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves, variant=kw.get("variant", 0))
    hs, g, errs = _run_ranks(pts, cfg.N, cfg.D, cfg.T, cfg.halves, world, cuda_device, **kw)
    assert errs == [None] * world, errs
    pairs = 0
    for h in hs:   # every rank holds the global result
        compare_all(h, ref, cfg.halves, cfg.D)
        st = h.stats()
        assert (st["tests"], st["votes"], st["leaves"]) == (ref.tests, ref.votes, ref.leaves.shape[0])
        pairs += st["pairs"]
    if "mem_budget" in kw:   # tail_depth 6 has no level D-5 lists, so fewer ranges
        assert min(h.stats()["ranges"] for h in hs) > (2 if kw.get("tail_depth") == 6 else 4) * cfg.D
    for h in hs:
        h.close()
    g.close()


@pytest.mark.parametrize("seed", range(6))
def test_multirank_random(seed, cuda_device):
    rng = np.random.default_rng(900 + seed)
    N = int(rng.choice([16, 64, 128, 200]))
    D = int(rng.integers(2, 9))
    T = int(rng.choice([2, 5, 12]))
    world = int(rng.integers(2, 5))
    pts = synth.random_scene(4000 + seed, N, max_lines=4, max_noise=int(rng.choice([100, 1500])))
    ref = oracle.detect(pts, N, D, T, AB)
    hs, g, errs = _run_ranks(pts, N, D, T, AB, world, cuda_device)
    assert errs == [None] * world, errs
    for h in hs:
        compare_all(h, ref, AB, D)
        h.close()
    g.close()


def test_multirank_error_flag_is_collective(cuda_device):
    """One rank holds an out-of-range point: every rank fails with HHT_ERANGE."""
    pts = synth.random_scene(7, 64, max_noise=200).copy()
    pts[-1] = (64, 3)                    # lands on the last rank
    hs, g, errs = _run_ranks(pts, 64, 6, 5, AB, 2, cuda_device)
    assert all(isinstance(e, hht.HHTError) and e.name == "HHT_ERANGE" for e in errs), errs
    for h in hs:
        h.close()
    g.close()


@pytest.mark.parametrize("cid,budget", [(3, 0), (3, 24 << 20), (5, 40 << 30)])
def test_multirank_digest(cid, budget, cuda_device):
    """Configs 3 and 5 on 2 ranks (points sharded), the fused tail's grid allreduce deferred onto a
    second stream behind the next range (config 5: 40 GiB per rank, both ranks share the one GPU,
    several ranges; config 3 with a 24 MiB budget runs in nested depth-first ranges). Every level's
    records and the leaves hash to the oracle's digest on both ranks."""
    import hashlib
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"c{cid}_digest.json")))
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    hs, g, errs = _run_ranks(pts, cfg.N, cfg.D, cfg.T, cfg.halves, 2, cuda_device, mem_budget=budget)
    assert errs == [None, None], errs
    for h in hs:
        for half in (1, 2):
            for lev in range(cfg.D + 1):
                arr = np.ascontiguousarray(h.level(0, half, lev).astype("<u4"))
                assert hashlib.sha256(arr.tobytes()).hexdigest() == gold["level_sha256"][f"{half}/{lev}"], (half, lev)
        lv = np.ascontiguousarray(h.leaves(-1).astype("<u4"))
        assert hashlib.sha256(lv.tobytes()).hexdigest() == gold["leaves_sha256"]
        st = h.stats()
        assert (st["tests"], st["votes"]) == (gold["tests"], gold["votes"])
    if budget and cid == 3:
        assert min(h.stats()["ranges"] for h in hs) > 2 * cfg.D
    for h in hs:
        h.close()
    g.close()


@pytest.mark.parametrize("budget", [0, 256 << 10])
def test_multirank_packed_leaf_sink(budget, cuda_device):
    """The packed leaf sink on 2 ranks (depth-first ranges under a small budget, where each range's
    leaf-grid work is deferred behind the next range): every rank streams the global leaves, in
    order, equal to the oracle's."""
    from tests.test_gpu_parity import _unpack_rows
    cfg = synth.CONFIGS[2]
    pts, _ = synth.config_image(2)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    want = ref.leaves.shape[0]
    sinks = {}

    def setup(h):
        sinks[id(h)] = np.zeros(want + 3, dtype=np.uint64)
        h.set_leaf_sink_packed(sinks[id(h)])

    hs, g, errs = _run_ranks(pts, cfg.N, cfg.D, cfg.T, cfg.halves, 2, cuda_device, setup=setup, mem_budget=budget)
    assert errs == [None, None], errs
    for h in hs:
        st = h.stats()
        assert st["leaves_streamed"] == st["leaves"] == want
        rows = _unpack_rows(sinks[id(h)][:want], h.tree_offsets(), 2, cfg.halves)
        assert np.array_equal(rows, h.leaves(-1))       # the streamed rows are the result ...
        compare_all(h, ref, cfg.halves, cfg.D)           # ... and the result is the oracle's
        h.close()
    g.close()
