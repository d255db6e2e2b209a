"""Pins of the oracle's detector with solution()'s point removal ON (oracle_detect_removal;
PAPER.md:178-204): against an independently written greedy post-pass over
the removal-off candidates (emit a candidate leaf, in depth-first order, iff
its voters not yet removed exceed the threshold, then remove them), with supports recomputed from the
literal 4-bit code (oracle.code); plus the removal invariants (disjoint supports, live votes)."""
import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import synth

MIXED = lambda code: code not in (0b0000, 0b1111)  # noqa: E731


def greedy(points, N, D, T, half):
    ref = oracle.detect(points, N, D, T, half)
    removed = set()
    out, sup = [], []
    for h, i, j, _ in ref.leaves.tolist():
        s = [p for p, (x, y) in enumerate(points.tolist()) if MIXED(oracle.code(x, y, half, N, D, D, i, j))]
        live = [p for p in s if p not in removed]
        if len(live) > T:
            out.append((h, i, j, len(live)))
            sup.append(set(live))
            removed.update(live)
    return out, sup


@pytest.mark.parametrize("seed", range(40))
def test_removal_equals_greedy_post_pass(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.choice([8, 13, 16, 32, 64]))
    D = int(rng.integers(2, 7))
    T = int(rng.choice([1, 2, 3, 5, 8]))
    pts = synth.random_scene(200 + seed, N, max_lines=3, max_noise=int(rng.choice([5, 40, 120])))
    for half in (oracle.ALPHA, oracle.BETA):
        lines, sup = oracle.detect_removal(pts, N, D, T, half)
        want, want_sup = greedy(pts, N, D, T, half)
        assert [tuple(r) for r in lines.tolist()] == want
        got_sup = [set() for _ in range(len(lines))]
        for li, p in sup.tolist():
            got_sup[li].add(p)
        assert got_sup == want_sup


@pytest.mark.parametrize("cid", [1, 2])
def test_removal_invariants(cid):
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    ref = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    lines, sup = oracle.detect_removal(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    cand = {(h, i, j): v for h, i, j, v in ref.leaves.tolist()}
    for k, (h, i, j, v) in enumerate(lines.tolist()):
        assert (h, i, j) in cand and v <= cand[(h, i, j)] and v > cfg.T      # emitted leaves are candidates
        members = sup[sup[:, 0] == k, 1]
        assert len(members) == v                                            # live votes = support size
    for half in (oracle.ALPHA, oracle.BETA):
        idx = [k for k, r in enumerate(lines.tolist()) if r[0] == half]
        pts_used = sup[np.isin(sup[:, 0], idx), 1]
        assert len(pts_used) == len(set(pts_used.tolist()))                 # disjoint supports
    assert 0 < lines.shape[0] < ref.leaves.shape[0]
