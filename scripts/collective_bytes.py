"""Collective payload of a multi-rank detection per level, from an oracle digest's visited counts
(tests/golden/c<cfg>_digest.json), for the default schedule (fused tail at level D-5):
  - after the root count pass and after each count-ahead list pass at levels 0 .. D-7, one allreduce
    of the children's votes of the next frontier: 16 B per split region of levels 0 .. D-6;
  - after each fused-tail range, one allreduce of the 16x16 leaf grids of all 4 children of every
    split level-(D-5) region: 4 KiB per such region (overlapped with the next range on a second stream);
  - 8 B per depth-first range (agreement on the range end) and a few words per call.
The payload does not depend on W; a ring allreduce moves 2 (W-1)/W of it per rank each way.

    python scripts/collective_bytes.py --config 5
"""
import argparse
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--bw", type=float, default=725.0, help="all-reduce bus bandwidth GB/s (B200_PROFILING.md, 8 ranks)")
    a = ap.parse_args()
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"c{a.config}_digest.json")))
    D = g["D"]
    halves = [h for h in (1, 2) if g["halves"] & h]
    visited = [sum(g["level_count"][f"{h}/{l}"] for h in halves) for l in range(D + 1)]
    split = [visited[l + 1] // 4 for l in range(D)]           # split regions at level l
    rows = []
    for l in range(D - 5):                                     # vote allreduces for frontiers 0 .. D-6
        rows.append((f"votes of the children of the level-{l} frontier", 16 * split[l]))
    rows.append((f"leaf grids of the level-{D - 4} regions (4 x 1 KiB per split level-{D - 5} region)",
                 4096 * split[D - 5]))
    total = sum(b for _, b in rows)
    print(f"| collective (config {a.config}, payload per detection) | bytes |")
    print("|---|---|")
    for name, b in rows:
        print(f"| {name} | {b:,} |")
    print(f"| total | {total:,} |")
    print()
    print("| W | bytes sent per rank (ring, 2(W-1)/W x payload) | time at the measured 8-rank bus bandwidth (725 GB/s) |")
    print("|---|---|---|")
    for W in (2, 4, 8):
        per = 2 * (W - 1) / W * total
        print(f"| {W} | {per / 1e9:.2f} GB | {per / (a.bw * 1e9) * 1e3:.2f} ms |")


if __name__ == "__main__":
    main()
