"""Phase trace of the one-block latency kernel k_small on config 1: globaltimer stamps written by
thread 0 at each phase boundary (pass 1, the children scan, pass 2 per level) of the last launch.
Needs the experiment build:

    bash scripts/build_variant.sh strace -DHHT_SMALL_TRACE && python scripts/small_trace.py
"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1007_0547_b200 import hht, synth
lib = hht.load(os.path.join(os.path.dirname(hht.LIB_PATH), "libhht_strace.so"))
cfg = synth.CONFIGS[1]
pts, _ = synth.config_image(1)
h = hht.HHT(halves=cfg.halves, latency_path=1, profile=True)
d = torch.from_numpy(pts).cuda()
for _ in range(20):
    h.detect(d, cfg.N, cfg.D, cfg.T)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 512)()
print("rc", lib.hht_debug_small_trace(buf))
t = list(buf)
t0 = t[0]
print("start->roots", (t[1] - t0) / 1e3, "us; total", (t[7] - t0) / 1e3)
for l in range(cfg.D):
    b = 8 + 8 * l
    print(l, "pass1", (t[b + 1] - t[b]) / 1e3, "children", (t[b + 2] - t[b + 1]) / 1e3,
          "pass2", (t[b + 6] - t[b + 2]) / 1e3 if l + 1 < cfg.D else -1)
