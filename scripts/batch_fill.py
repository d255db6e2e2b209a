"""Raster batch fill of the fused tail: for every level-(D-4) region whose grid the fused tail
rasters (the 4 children of each split level-(D-5) region), its list length is its vote count, and
the tail rasters it in ceil(votes / B) batches of B = 32 x ITEMS lane slots (ITEMS = 13, the
kernel's HHT_FUSED_ITEMS; --items to model another build). Prints the fill factor (lines /
lane slots) and the split of batches by item count per lane, from the level records of one detection.

    python scripts/batch_fill.py --config 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--items", type=int, default=13, help="lines per lane per raster batch (HHT_FUSED_ITEMS)")
a = ap.parse_args()
BATCH = 32 * a.items
cfg = synth.CONFIGS[a.config]
if cfg.images > 1:
    pts, offs = synth.config_batch(a.config, 16)
else:
    pts, _ = synth.config_image(a.config)
    offs = np.array([0, len(pts)])
h = hht.HHT(halves=cfg.halves)
h.detect_batch(torch.from_numpy(pts).cuda(), offs, cfg.N, cfg.D, cfg.T)
L = cfg.D - 4
v = []
for img in range(len(offs) - 1):
    for half in (hht.ALPHA, hht.BETA):
        if not (cfg.halves & half):
            continue
        r = h.level(img, half, L)
        v.append(r[:, 2].astype(np.int64))
v = np.concatenate(v)
v = v[v > 0]
batches = (v + BATCH - 1) // BATCH
slots = batches.sum() * BATCH
print(f"config {a.config}: level {L} regions with lines {len(v)}, lines {v.sum()}, batches {batches.sum()}, "
      f"fill {v.sum() / slots:.3f}")
last = v - (batches - 1) * BATCH                       # lines in each region's last batch
items = (last + 31) // 32
full = (batches - 1).sum()
print("full batches", int(full), "last-batch items/lane histogram:",
      {int(k): int((items == k).sum()) for k in range(1, a.items + 1)})
print("fill if the last batch ran ceil(n/32) items:",
      f"{v.sum() / (32 * (a.items * full + items.sum())):.3f}")
