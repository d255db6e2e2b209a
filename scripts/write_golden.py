"""Write full-size parity digests of the CPU oracle for a BASELINE config.

    python scripts/write_golden.py --config 3 [--workers 6] [--split-level 2]

Calls only oracle/ and the seeded generator (paper_1007_0547_b200/synth.py). Output:
tests/golden/c<cfg>_digest.json with, per (half, level), the record count and the sha256 of the
uint32 little-endian array of (a, c, votes) triplets of every image concatenated in image order;
the sha256 of the leaves as uint32 (image, half, i, j, votes) rows; and the tests/votes totals.

Large trees are split into independent level-k subtrees (oracle.detect_subtree): a region's votes
do not depend on which ancestor list it was tested from (containment), so the
concatenation of the subtrees' records in depth-first order equals the plain depth-first run.
Levels < k come from a plain oracle.detect of depth k (region geometry at level l does not depend
on the leaf depth). Tests are recomputed from the records: E + 4 * sum of split votes per tree.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1007_0547_b200 import synth  # noqa: E402

_PTS = {}


def _points(cid, image):
    key = (cid, image)
    if key not in _PTS:
        _PTS.clear()
        _PTS[key] = synth.config_image(cid, image)[0]
    return _PTS[key]


def _subtree(args):
    cid, image, half, k, a, c = args
    cfg = synth.CONFIGS[cid]
    r = oracle.detect_subtree(_points(cid, image), cfg.N, cfg.D, cfg.T, half, k, a, c)
    return {lev: r.levels[(half, lev)] for lev in range(k, cfg.D + 1)}, r.leaves


def _tree_tasks(cid, image, half, k):
    cfg = synth.CONFIGS[cid]
    pts = _points(cid, image)
    kk = min(k, cfg.D)
    top = oracle.detect(pts, cfg.N, kk, cfg.T, half)
    levels = {lev: top.levels[(half, lev)] for lev in range(kk)}
    tasks = [(cid, image, half, kk, int(a), int(c)) for a, c, _ in top.levels[(half, kk)].tolist()]
    return levels, tasks


def tree_records(cid, image, half, k, pool):
    cfg = synth.CONFIGS[cid]
    levels, tasks = _tree_tasks(cid, image, half, k)
    parts = list(pool.map(_subtree, tasks)) if pool else list(map(_subtree, tasks))
    for lev in range(min(k, cfg.D), cfg.D + 1):
        arrs = [p[0][lev] for p in parts]
        levels[lev] = np.concatenate(arrs) if arrs else np.zeros((0, 3), np.uint32)
    leaves = [p[1] for p in parts]
    leaves = np.concatenate(leaves) if leaves else np.zeros((0, 4), np.uint32)
    return levels, leaves


def _whole_image(args):
    cid, image = args
    cfg = synth.CONFIGS[cid]
    pts = _points(cid, image)
    r = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
    return image, {h: {lev: r.levels[(h, lev)] for lev in range(cfg.D + 1)} for h in (1, 2) if cfg.halves & h}, r.leaves


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--split-level", type=int, default=2)
    ap.add_argument("--images", type=int, default=None)
    a = ap.parse_args()
    cid = a.config
    cfg = synth.CONFIGS[cid]
    B = cfg.images if a.images is None else a.images
    t0 = time.time()
    hashes = {}
    counts = {}
    leaf_rows = []
    tests = votes = 0
    halves = [h for h in (1, 2) if cfg.halves & h]
    per_level = {(h, lev): [] for h in halves for lev in range(cfg.D + 1)}
    with ProcessPoolExecutor(a.workers) as pool:
        if B > 1:
            results = sorted(pool.map(_whole_image, [(cid, b) for b in range(B)]), key=lambda r: r[0])
            for image, lv, leaves in results:
                for h in halves:
                    for lev in range(cfg.D + 1):
                        per_level[(h, lev)].append(lv[h][lev])
                if leaves.shape[0]:
                    leaf_rows.append(np.concatenate([np.full((leaves.shape[0], 1), image, np.uint32), leaves], 1))
        else:
            for h in halves:
                lv, leaves = tree_records(cid, 0, h, a.split_level, pool)
                for lev in range(cfg.D + 1):
                    per_level[(h, lev)].append(lv[lev])
                if leaves.shape[0]:
                    leaf_rows.append(np.concatenate([np.zeros((leaves.shape[0], 1), np.uint32), leaves], 1))
    for (h, lev), arrs in per_level.items():
        arr = np.ascontiguousarray(np.concatenate(arrs).astype("<u4"))
        hashes[f"{h}/{lev}"] = hashlib.sha256(arr.tobytes()).hexdigest()
        counts[f"{h}/{lev}"] = int(arr.shape[0])
        votes += int(arr[:, 2].astype(np.int64).sum())
        if lev < cfg.D:
            tests += 4 * int(arr[:, 2][arr[:, 2] > cfg.T].astype(np.int64).sum())
        if lev == 0:
            tests += int(arr[:, 2].astype(np.int64).sum())
    leaves = np.concatenate(leaf_rows) if leaf_rows else np.zeros((0, 5), np.uint32)
    # sort leaves by image then half, keeping depth-first order inside a tree
    order = np.lexsort((np.arange(leaves.shape[0]), leaves[:, 1], leaves[:, 0]))
    leaves = np.ascontiguousarray(leaves[order].astype("<u4"))
    out = {
        "source": "written by scripts/write_golden.py: oracle/ (plain C DFS, PAPER.md §3) on the seeded "
                  f"generator's config {cid} ({cfg.text}); calls nothing but oracle/ and synth.py",
        "config": cid, "images": B, "N": cfg.N, "D": cfg.D, "T": cfg.T, "halves": cfg.halves,
        "level_sha256": hashes, "level_count": counts,
        "leaves_sha256": hashlib.sha256(leaves.tobytes()).hexdigest(), "leaves": int(leaves.shape[0]),
        "tests": tests, "votes": votes, "oracle_seconds": round(time.time() - t0, 1),
    }
    path = os.path.join(ROOT, "tests", "golden", f"c{cid}_digest.json" if a.images is None else
                        f"c{cid}_first{B}_digest.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, out["oracle_seconds"], "s")


if __name__ == "__main__":
    main()
