"""Write the digest of the oracle's depth-first detector with solution()'s point removal ON
(oracle.detect_removal = oracle_detect_removal) for a BASELINE config.

    python scripts/write_golden_removal.py --config 3

Calls only oracle/ and the seeded generator (paper_1007_0547_b200/synth.py); one process per half
(the removal-on walk of one tree is sequential). Output: tests/golden/c<cfg>_removal_digest.json with
the emitted lines (half, i, j, live votes) as uint32 rows in emission order (ALPHA tree first) and
their sha256, and the sha256 of the supports as uint32 (line index, point index) rows sorted by line
then point (each point belongs to at most one line per tree).
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


def _half(args):
    cid, half = args
    cfg = synth.CONFIGS[cid]
    pts, _ = synth.config_image(cid)
    lines, sup = oracle.detect_removal(pts, cfg.N, cfg.D, cfg.T, half)
    return half, lines, sup


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    assert cfg.images == 1, "single-image configs"
    t0 = time.time()
    halves = [h for h in (1, 2) if cfg.halves & h]
    with ProcessPoolExecutor(len(halves)) as pool:
        res = sorted(pool.map(_half, [(a.config, h) for h in halves]), key=lambda r: r[0])
    lines, sups = [], []
    base = 0
    for half, ln, sp in res:
        lines.append(ln)
        if sp.shape[0]:
            sp = sp.astype(np.int64).copy()
            sp[:, 0] += base
            sups.append(sp)
        base += ln.shape[0]
    L = np.ascontiguousarray(np.concatenate(lines).astype("<u4")) if lines else np.zeros((0, 4), "<u4")
    S = np.concatenate(sups) if sups else np.zeros((0, 2), np.int64)
    S = np.ascontiguousarray(S[np.lexsort((S[:, 1], S[:, 0]))].astype("<u4"))
    out = {
        "source": "written by scripts/write_golden_removal.py: oracle_detect_removal (plain C depth-first "
                  f"detector with solution()'s point removal ON, PAPER.md:178-204) on config {a.config} "
                  f"({cfg.text}); calls nothing but oracle/ and synth.py",
        "config": a.config, "N": cfg.N, "D": cfg.D, "T": cfg.T, "halves": cfg.halves,
        "lines": int(L.shape[0]), "lines_sha256": hashlib.sha256(L.tobytes()).hexdigest(),
        "lines_per_half": {str(h): int(ln.shape[0]) for h, ln, _ in res},
        "live_votes_total": int(L[:, 3].astype(np.int64).sum()) if L.shape[0] else 0,
        "support": int(S.shape[0]), "support_sha256": hashlib.sha256(S.tobytes()).hexdigest(),
        "first_lines": L[:8].tolist(), "oracle_seconds": round(time.time() - t0, 1),
    }
    path = os.path.join(ROOT, "tests", "golden", f"c{a.config}_removal_digest.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, out["lines"], out["support"], out["oracle_seconds"], "s")


if __name__ == "__main__":
    main()
