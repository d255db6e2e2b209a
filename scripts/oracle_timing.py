"""Full-config timing of the CPU oracle on the machine's own cores (SURVEY.md §8(d) "Oracle timing plan").

    python scripts/oracle_timing.py [--single 1,2,3] [--all-cores 3,4,5] [--out profiles/r02_oracle_timing.md]

Times the oracle AS IT STANDS (oracle/, plain C -O2, no OpenMP): single-thread = one oracle_detect call per
image on one core; all-cores = one process per core (os.cpu_count()) over independent work units
(single-image configs: the level-k subtrees of every tree, as scripts/write_golden.py splits them; batch
configs: whole images). tests = the paper's code evaluations (E + 4 x the votes of every split region, per
tree), recomputed from the records and checked against the oracle-written digest in tests/golden/ where one
exists. Prints lscpu's model name and the core count. The oracle is test infrastructure: this script only
measures it (the baseline bench.py's cpu_baseline samples from the same code path).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import oracle  # noqa: E402
from paper_1007_0547_b200 import synth  # noqa: E402
import write_golden as wg  # noqa: E402  (its subtree / whole-image work units)


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def tests_of(levels_by_tree, E_by_tree, T, D):
    """E + 4 * sum of split votes, summed over trees; levels[l] = (a, c, votes) rows."""
    t = 0
    for key, levels in levels_by_tree.items():
        t += E_by_tree[key]
        for lev in range(D):
            v = levels[lev][:, 2].astype(np.int64)
            t += 4 * int(v[v > T].sum())
    return t


def single_thread(cid):
    cfg = synth.CONFIGS[cid]
    tests = 0
    secs = 0.0
    for b in range(cfg.images):
        pts, _ = synth.config_image(cid, b)
        t0 = time.perf_counter()
        r = oracle.detect(pts, cfg.N, cfg.D, cfg.T, cfg.halves)
        secs += time.perf_counter() - t0
        tests += r.tests
    return secs, tests, 1


def all_cores(cid, workers, split_level):
    cfg = synth.CONFIGS[cid]
    halves = [h for h in (1, 2) if cfg.halves & h]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(workers) as pool:
        if cfg.images > 1:
            res = list(pool.map(wg._whole_image, [(cid, b) for b in range(cfg.images)]))
            lv = {(img, h): levels[h] for img, levels, _ in res for h in halves}
            E = {(b, h): synth.config_image(cid, b)[0].shape[0] for b in range(cfg.images) for h in halves}
        else:
            lv, E = {}, {}
            n = synth.config_image(cid, 0)[0].shape[0]
            for h in halves:
                levels, _ = wg.tree_records(cid, 0, h, split_level, pool)
                lv[(0, h)] = levels
                E[(0, h)] = n
    secs = time.perf_counter() - t0
    return secs, tests_of(lv, E, cfg.T, cfg.D), workers


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--single", default="1,2,3")
    ap.add_argument("--all-cores", default="3,4")
    ap.add_argument("--split-level", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_timing.md"))
    a = ap.parse_args()
    oracle.build()
    ncpu = os.cpu_count() or 1
    model = cpu_model()
    rows = []
    runs = [("single", int(c)) for c in a.single.split(",") if c] + \
           [("all", int(c)) for c in a.all_cores.split(",") if c]
    for mode, cid in runs:
        cfg = synth.CONFIGS[cid]
        secs, tests, thr = single_thread(cid) if mode == "single" else all_cores(cid, ncpu, a.split_level)
        gold = os.path.join(ROOT, "tests", "golden", f"c{cid}_digest.json")
        check = "-"
        if os.path.exists(gold):
            check = "= digest" if json.load(open(gold))["tests"] == tests else "DIFFERS from digest"
        rows.append((cid, cfg.text, mode, thr, secs, tests, tests / secs, 1e3 * secs / cfg.images, check))
        print(rows[-1], flush=True)
    with open(a.out, "w") as f:
        f.write("# Oracle (plain C, oracle/ as it stands) on the GPU box's host cores, full configs\n\n")
        f.write(f"CPU: {model}; os.cpu_count() = {ncpu}. Single-thread: one oracle_detect per image on one core. "
                f"All cores: one process per core over independent work units (level-{a.split_level} subtrees of "
                "each tree for one-image configs, whole images for config 4). Wall-clock seconds of the whole "
                "config; tests = the paper's code evaluations (checked against the oracle-written digest).\n\n")
        f.write("| config | mode | threads | seconds | tests | tests/s | ms per image | tests check |\n")
        f.write("|---|---|---|---|---|---|---|---|\n")
        for cid, text, mode, thr, secs, tests, tps, mspi, check in rows:
            f.write(f"| C{cid} | {'single thread' if mode == 'single' else 'all cores'} | {thr} | {secs:.2f} | "
                    f"{tests:.4g} | {tps:.3g} | {mspi:.4g} | {check} |\n")
    print(a.out)


if __name__ == "__main__":
    main()
