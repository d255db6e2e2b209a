import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1007_0547_b200 import hht, synth
cfg = synth.CONFIGS[5]
pts, _ = synth.config_image(5)
offs = np.array([0, len(pts)], dtype=np.int64)
host = torch.from_numpy(pts).pin_memory().numpy()
d = torch.from_numpy(pts).cuda()
h = hht.HHT(halves=cfg.halves, profile=False)
h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)
n = h.stats()["leaves"]
buf = torch.empty((n + 1024, 5), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
def t(f, k=3):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(1e3*(time.perf_counter()-t0))
    return [round(x, 1) for x in ts]
print("device pts, no sink        ", t(lambda: h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)), "dev ms", round(h.stats()["ms"],1))
print("host pts, no sink          ", t(lambda: h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)), "dev ms", round(h.stats()["ms"],1))
print("host pts + leaves_into     ", t(lambda: (h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T), h.leaves_into(buf))))
h.set_leaf_sink(buf)
print("host pts + sink            ", t(lambda: h.detect_batch(host, offs, cfg.N, cfg.D, cfg.T)), "dev ms", round(h.stats()["ms"],1), h.stats()["leaves_streamed"])
print("device pts + sink          ", t(lambda: h.detect_batch(d, offs, cfg.N, cfg.D, cfg.T)), "dev ms", round(h.stats()["ms"],1))
t0=time.perf_counter(); torch.from_numpy(buf).cuda(); torch.cuda.synchronize(); print("H2D 1.2GB ms", 1e3*(time.perf_counter()-t0))
x = torch.empty((n+1024)*5, dtype=torch.int32, device='cuda')
hb = torch.from_numpy(buf.view(np.int32).reshape(-1))
torch.cuda.synchronize(); t0=time.perf_counter(); hb.copy_(x, non_blocking=True); torch.cuda.synchronize(); print("D2H 1.2GB ms", 1e3*(time.perf_counter()-t0))
