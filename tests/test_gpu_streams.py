"""Stream ordering at the boundary (include/hht.h hht_opts.stream / hht_set_stream): a detection on
device input produced by work still queued on the caller's current stream must see that input. The
producer here is a copy queued behind a ~20 ms sleep kernel on a side stream; the binding passes
torch's current stream to the library (borrowed), so no host synchronisation is needed and none is
done. Without the ordering the library would read the zero-filled buffer."""
import numpy as np
import pytest

import oracle
from paper_1007_0547_b200 import hht, synth
from tests.hht_compare import compare_all

pytestmark = pytest.mark.gpu


def test_detect_waits_for_producer_on_side_stream(cuda_device):
    import torch
    pts = synth.random_scene(515, 64, max_lines=3, max_noise=200)
    src = torch.from_numpy(pts).to(cuda_device)
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    h = hht.HHT(halves=hht.ALPHA | hht.BETA, latency_path=2)
    s = torch.cuda.Stream(cuda_device)
    with torch.cuda.stream(s):
        torch.cuda._sleep(40_000_000)        # ~20 ms of device time before the producer copy
        dst.copy_(src, non_blocking=True)
        h.detect(dst, 64, 6, 4)
    ref = oracle.detect(pts, 64, 6, 4, hht.ALPHA | hht.BETA)
    compare_all(h, ref, hht.ALPHA | hht.BETA, 6)
    # back on the default stream: the ctx follows torch's current stream again
    h.detect(src, 64, 6, 4)
    compare_all(h, ref, hht.ALPHA | hht.BETA, 6)


def test_detect_image_waits_for_producer_on_side_stream(cuda_device):
    """detect_image on a CUDA tensor must be ordered after the image's producer."""
    import torch
    N = 96
    rng = np.random.default_rng(5)
    img = (rng.random((N, N)) < 0.1).astype(np.uint8) * 200
    src = torch.from_numpy(img).to(cuda_device)
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    h_dev = hht.HHT(halves=hht.ALPHA | hht.BETA)
    h_host = hht.HHT(halves=hht.ALPHA | hht.BETA)
    h_host.detect_image(img, 100, 7, 3)
    s = torch.cuda.Stream(cuda_device)
    with torch.cuda.stream(s):
        torch.cuda._sleep(40_000_000)
        dst.copy_(src, non_blocking=True)
        h_dev.detect_image(dst, 100, 7, 3)
    ea, eb = h_dev.edges()
    ha, hb = h_host.edges()
    assert ea.shape[0] + eb.shape[0] > 0
    assert np.array_equal(ea, ha) and np.array_equal(eb, hb)
    assert np.array_equal(h_dev.leaves(0), h_host.leaves(0))


def test_borrowed_stream_opt(cuda_device):
    """hht_opts.stream: the ctx enqueues on the caller's stream from creation on."""
    import torch
    pts = synth.random_scene(516, 128, max_lines=3, max_noise=500)
    s = torch.cuda.Stream(cuda_device)
    h = hht.HHT(halves=hht.ALPHA | hht.BETA, stream=s.cuda_stream, latency_path=2)
    host = np.ascontiguousarray(pts)
    h.detect(host, 128, 7, 5)                 # host input: no rebinding; runs on s
    ref = oracle.detect(pts, 128, 7, 5, hht.ALPHA | hht.BETA)
    compare_all(h, ref, hht.ALPHA | hht.BETA, 7)
