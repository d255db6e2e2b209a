"""CPU-only checks of the boundary and host logic (no compute calls without a GPU)."""
import ctypes
import re
from fractions import Fraction
import os
import json

import numpy as np
import pytest

from paper_1007_0547_b200 import build as hbuild
from paper_1007_0547_b200 import hht, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    hbuild.build()
    return hht.load()


def test_library_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "hht.h")).read()
    names = set(re.findall(r"\b(hht_[a-z_]+)\s*\(", hdr))
    assert names == set(hht.EXPORTS), names ^ set(hht.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", hht.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings(lib):
    assert hht.version().startswith("hht ") and "sm_100a" in hht.version()
    for k, v in hht.STATUS.items():
        assert lib.hht_status_str(k).decode() == v


def test_default_opts(lib):
    o = hht.Opts()
    assert lib.hht_default_opts(ctypes.byref(o)) == 0
    assert (o.world, o.rank, o.halves, o.record_levels, o.mem_budget) == (1, 0, 3, 1, 0)


def test_create_without_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(hht.HHTError) as e:
        hht.HHT()
    assert e.value.name == "HHT_ECUDA"


def test_null_context_is_einval(lib):
    import ctypes as C
    cnt = C.c_int64(0)
    assert lib.hht_detect(None, None, 0, 8, 3, 1) == 1
    assert lib.hht_result_leaves(None, 0, None, 0, C.byref(cnt)) == 1
    lib.hht_destroy(None)   # NULL-safe


def test_leaf_bounds_spec_example():
    """n = n_cells = 8, first cell -> m in [-1,-0.75], b in [-8,-5]."""
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_spec_examples.json")))["leaf_params"]
    assert hht.leaf_bounds(g["i"], g["j"], g["N"], g["D"]) == (
        Fraction(g["m_lo"]), Fraction(g["m_hi"]), Fraction(g["b_lo"]), Fraction(g["b_hi"]))
    # widths 2/2^D and 3N/2^D everywhere
    m0, m1, b0, b1 = hht.leaf_bounds(5, 7, 8, 3)
    assert m1 - m0 == Fraction(2, 8) and b1 - b0 == Fraction(24, 8)


def test_generator_deterministic_and_in_range():
    a, ta = synth.config_image(2)
    b, tb = synth.config_image(2)
    assert np.array_equal(a, b) and ta == tb
    assert a.dtype == np.int32 and a.shape == (17107, 2) and a.min() >= 0 and a.max() < 512
    assert len(ta) == 20 and {t.half for t in ta} == {1, 2}


def test_generator_line_points_lie_on_their_lines():
    cfg = synth.CONFIGS[1]
    pts, truth = synth.config_image(1)
    s = set(map(tuple, pts.tolist()))
    for t in truth:
        hits = 0
        for x in range(cfg.N):
            u = (t.A * x + t.Q + (1 << 15)) // (1 << 16)
            if (x, u) in s:
                hits += 1
        assert hits >= t.k


def test_shard_partition():
    for n in [0, 1, 7, 100, 12345]:
        for w in [1, 2, 3, 8]:
            parts = [synth.shard(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
