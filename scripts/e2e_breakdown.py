"""Where the end-to-end time of a config-5 call goes: device-resident points vs pinned host points,
with and without the leaf sink (median of --reps wall-clock calls after warm-up).

    python scripts/e2e_breakdown.py
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1007_0547_b200 import hht, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
pts, _ = synth.config_image(a.config)
offs = np.array([0, len(pts)])
dev = torch.from_numpy(pts).cuda()
host = torch.from_numpy(pts).pin_memory().numpy()
h = hht.HHT(halves=cfg.halves)


def wall(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts), h.stats()["ms"]


print("device points, no sink: wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(dev, offs, cfg.N, cfg.D, cfg.T)))
print("host points,   no sink: wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)))
n = h.stats()["leaves"]
buf = torch.empty((int(n * 1.1) + 1024, 5), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
h.set_leaf_sink(buf)
print("device points, sink:    wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(dev, offs, cfg.N, cfg.D, cfg.T)))
print("host points,   sink:    wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)))
st = h.stats()
print("leaves", st["leaves"], "streamed", st["leaves_streamed"], "ranges", st["ranges"])
# the final-range cut alone: a sink with no room (the driver cuts the last range, copies nothing)
h.set_leaf_sink(buf[:0])
print("device points, sink cap 0 (cut, no copies): wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(dev, offs, cfg.N, cfg.D, cfg.T)))
print("ranges", h.stats()["ranges"])
pk = torch.empty(int(n * 1.1) + 1024, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
h.set_leaf_sink_packed(pk)
print("device points, packed sink: wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(dev, offs, cfg.N, cfg.D, cfg.T)))
print("host points,   packed sink: wall %.1f ms, device %.1f ms" % wall(lambda: h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)))
h.set_leaf_sink(None)
