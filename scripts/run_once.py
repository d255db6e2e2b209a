"""Run `--reps` detections of one config through the C ABI (for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--images", type=int, default=None)
ap.add_argument("--budget", type=int, default=0)
ap.add_argument("--tail", type=int, default=0)
ap.add_argument("--prefetch", type=int, default=0)
ap.add_argument("--variant", type=int, default=0, help="0 exact, 1 FHT circumcircle")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if cfg.images > 1:
    pts, offs = synth.config_batch(a.config, a.images)
else:
    pts, _ = synth.config_image(a.config)
    offs = np.array([0, len(pts)])
d = torch.from_numpy(pts).cuda()
h = hht.HHT(halves=cfg.halves, mem_budget=a.budget, profile=True, tail_depth=a.tail, prefetch=a.prefetch, variant=a.variant)
for _ in range(a.reps):
    h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)
st = h.stats()
prof = h.profile()
print({k: round(v["ms"], 2) for k, v in prof.items() if v["ms"] > 0})
print({k: st[k] for k in ("tests", "votes", "leaves", "pairs", "ranges", "ms", "int_bits")})
# per-launch algorithmic bytes, to pair with an ncu capture of the same launch (ncu -k regex:k_tail -c 1
# is the first "tail" launch; ncu -k regex:k_pass -s S -c 1 is k_pass launch S counting the root count)
log = h.launches()
by = {}
for cls, b, ms in log:
    by.setdefault(cls, []).append((b, ms))
for cls in ("count", "write", "tail", "split", "gather", "other"):
    xs = by.get(cls, [])
    if xs:
        print(cls, "launches", len(xs), "first bytes", xs[0][0], "bytes[:16]", [b for b, _ in xs[:16]])
        print(cls, "ms[:16]", [round(m, 3) for _, m in xs[:16]],
              "GB/s[:16]", [round(b / m / 1e6) if m > 0 else 0 for b, m in xs[:16]])
