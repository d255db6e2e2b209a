"""Per-launch log of one detection (opts.profile): class, algorithmic bytes, CUDA-event ms, GB/s.
    python scripts/launch_log.py --config 5 [--min-ms 0.2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--min-ms", type=float, default=0.2)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if cfg.images > 1:
    pts, offs = synth.config_batch(a.config)
else:
    pts, _ = synth.config_image(a.config)
    offs = np.array([0, len(pts)])
h = hht.HHT(halves=cfg.halves, profile=True)
d = torch.from_numpy(pts).cuda()
for _ in range(3):
    h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)
tot = 0.0
for i, (cls, b, ms) in enumerate(h.launches()):
    tot += ms
    if ms >= a.min_ms:
        print(f"{i:4d} {cls:8s} {ms:8.3f} ms {b / 1e9:8.3f} GB {b / 1e9 / (ms / 1e3) if ms else 0:8.0f} GB/s")
print("sum of launches", round(tot, 2), "ms; device", round(h.stats()["ms"], 2), "ms")
