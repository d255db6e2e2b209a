"""One removal post-pass (hht_result_lines) on a config, for ncu launch lists.
    python scripts/removal_profile.py --config 4"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if cfg.images > 1:
    pts, offs = synth.config_batch(a.config)
else:
    pts, _ = synth.config_image(a.config)
    offs = np.array([0, pts.shape[0]], dtype=np.int64)
h = hht.HHT(halves=cfg.halves)
d = torch.from_numpy(pts).cuda()
h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = h.lines().shape[0]
print("lines", n, "ms", 1e3 * (time.perf_counter() - t0))
