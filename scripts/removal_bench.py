"""Time of the removal post-pass (hht_result_lines, NEXT-1) on one B200 for configs 1-2 and the
Table-1-style scenes: support bitsets (candidates x points bits) + the per-tree sequential greedy.

    python scripts/removal_bench.py --out profiles/r01_removal.md
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402


def run(name, pts, N, D, T, halves, rows):
    h = hht.HHT(halves=halves)
    d = torch.from_numpy(pts).cuda()
    h.detect(d, N, D, T)
    det_ms = h.stats()["ms"]
    cand = h.leaves().shape[0]
    h.detect(d, N, D, T)                        # fresh result, then time the post-pass alone
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = h.lines().shape[0]
    ms = 1e3 * (time.perf_counter() - t0)
    rows.append((name, pts.shape[0], cand, n, det_ms, ms))
    print(rows[-1], flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for cid in (1, 2):
        cfg = synth.CONFIGS[cid]
        pts, _ = synth.config_image(cid)
        run(f"config{cid}", pts, cfg.N, cfg.D, cfg.T, cfg.halves, rows)
    for N in (32, 64, 128, 256):
        pts, _ = synth.scene(N, 5, max(4, N // 2 + N // 8), 1, max(1, N * N // 50), False, 0x7AB1E1, 100 * N + 1, 7)
        run(f"{N}x{N} scene (T=N/2)", pts, N, N.bit_length() - 1, max(4, N // 2), hht.ALPHA | hht.BETA, rows)
    lines = ["# solution() with point removal on one B200 (NEXT-1)", "",
             "Post-pass wall time of hht_result_lines (support bitsets + per-tree greedy, first request after "
             "a detect), beside the detection's device time. Emitted lines equal the oracle's literal "
             "depth-first detector with removal on (tests/test_gpu_removal.py).", "",
             "| input | points | candidate leaves | emitted lines | detect ms | removal post-pass ms |",
             "|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} | {r[4]:.2f} | {r[5]:.2f} |")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if a.out:
        open(a.out, "w").write(txt)


if __name__ == "__main__":
    main()
