"""Python binding of libhht.so (include/hht.h): argument marshalling only.

Every step of the method runs in the library's CUDA kernels; this module converts arrays to
pointers and results to numpy. There is no CPU fallback: if libhht.so is missing or fails to
load, importing/using this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np

ALPHA = 1
BETA = 2
EXACT = 0          # opts.variant: the paper's exact 4-bit corner-code test
FHT_CIRCLE = 1     # opts.variant: FHT circumcircle test (the paper's comparison)
FHT_CIRCLE_MB = 2  # opts.variant: the same circle in (m, b) units (reading R22)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhht.so")

STATUS = {0: "HHT_OK", 1: "HHT_EINVAL", 2: "HHT_ERANGE", 3: "HHT_EOVERFLOW", 4: "HHT_ENOMEM",
          5: "HHT_ECUDA", 6: "HHT_ENCCL", 7: "HHT_EMISMATCH", 8: "HHT_ESTATE"}

# names the header declares (tests check every one is exported)
EXPORTS = ["hht_default_opts", "hht_create", "hht_nccl_unique_id", "hht_detect", "hht_detect_batch",
           "hht_result_leaves", "hht_result_level", "hht_result_stats", "hht_result_profile",
           "hht_result_launches", "hht_timer_begin", "hht_timer_end", "hht_last_error", "hht_status_str",
           "hht_destroy", "hht_version", "hht_set_leaf_sink", "hht_group_create", "hht_group_destroy",
           "hht_detect_trees", "hht_detect_image", "hht_result_edges", "hht_result_lines", "hht_set_stream",
           "hht_result_line_points", "hht_set_leaf_sink_packed", "hht_result_tree_offsets"]

PROFILE_CLASSES = ["stage", "count", "write", "tail", "split", "gather", "other", "allreduce"]


class HHTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("halves", C.c_uint32),
                ("record_levels", C.c_uint32), ("force_int64", C.c_uint32), ("profile", C.c_uint32),
                ("tail_depth", C.c_uint32), ("prefetch", C.c_uint32), ("latency_path", C.c_uint32),
                ("variant", C.c_uint32),
                ("mem_budget", C.c_size_t),
                ("nccl_id", C.c_void_p), ("group", C.c_void_p), ("stream", C.c_void_p), ("nccl_comm", C.c_void_p),
                ("tail_units", C.c_uint32)]


class Leaf(C.Structure):
    _fields_ = [("image", C.c_int32), ("half", C.c_uint32), ("i", C.c_uint32), ("j", C.c_uint32),
                ("votes", C.c_uint32)]


class Stats(C.Structure):
    _fields_ = [("tests", C.c_uint64), ("votes", C.c_uint64), ("leaves", C.c_uint64), ("pairs", C.c_uint64),
                ("visited", C.c_uint64 * 64), ("split", C.c_uint64 * 64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("levels", C.c_uint32), ("int_bits", C.c_uint32),
                ("ranges", C.c_uint32), ("images", C.c_uint32), ("ms", C.c_double),
                ("leaves_streamed", C.c_uint64), ("latency_path", C.c_uint32), ("reserved", C.c_uint32)]


class Launch(C.Structure):
    _fields_ = [("cls", C.c_uint32), ("reserved", C.c_uint32), ("bytes", C.c_uint64), ("ms", C.c_double)]


class Profile(C.Structure):
    _fields_ = [("launches", C.c_uint64 * 8), ("ms", C.c_double * 8), ("bytes", C.c_uint64 * 8),
                ("ops", C.c_uint64 * 8)]


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libhht.so (raises if it is absent: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    p, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
    sig = {
        "hht_default_opts": ([p], C.c_int),
        "hht_create": ([p, p], C.c_int),
        "hht_nccl_unique_id": ([p, C.c_size_t], C.c_int),
        "hht_detect": ([p, p, i64, i32, i32, i64], C.c_int),
        "hht_detect_batch": ([p, p, p, i32, i32, i32, i64], C.c_int),
        "hht_result_leaves": ([p, i32, p, i64, p], C.c_int),
        "hht_result_level": ([p, i32, u32, i32, p, i64, p], C.c_int),
        "hht_result_stats": ([p, p], C.c_int),
        "hht_set_leaf_sink": ([p, p, i64], C.c_int),
        "hht_set_leaf_sink_packed": ([p, p, i64], C.c_int),
        "hht_result_tree_offsets": ([p, p, i64, p], C.c_int),
        "hht_group_create": ([p, i32], C.c_int),
        "hht_detect_trees": ([p, p, p, i32, i32, i32, i64], C.c_int),
        "hht_detect_image": ([p, p, i32, i32, i32, i64], C.c_int),
        "hht_result_edges": ([p, p, i64, p, p], C.c_int),
        "hht_result_lines": ([p, i32, p, i64, p], C.c_int),
        "hht_result_line_points": ([p, i32, p, i64, p], C.c_int),
        "hht_group_destroy": ([p], None),
        "hht_result_profile": ([p, p], C.c_int),
        "hht_result_launches": ([p, p, i64, p], C.c_int),
        "hht_timer_begin": ([p], C.c_int),
        "hht_timer_end": ([p, p], C.c_int),
        "hht_last_error": ([p], C.c_char_p),
        "hht_status_str": ([C.c_int], C.c_char_p),
        "hht_destroy": ([p], None),
        "hht_set_stream": ([p, p], C.c_int),
        "hht_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def version() -> str:
    return load().hht_version().decode()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load().hht_nccl_unique_id(buf, 128)
    if st:
        raise HHTError(st, "ncclGetUniqueId failed")
    return buf.raw


def leaf_bounds(i: int, j: int, N: int, D: int):
    """Exact (m_lo, m_hi, b_lo, b_hi) of leaf (i, j): m_i = -1 + 2i/2^D, b_j = -N + 3N j/2^D
    (include/hht.h conventions; SPEC.md:236-244 leaf_params)."""
    side = 1 << D
    m = lambda k: Fraction(-1) + Fraction(2 * k, side)  # noqa: E731
    b = lambda k: Fraction(-N) + Fraction(3 * N * k, side)  # noqa: E731
    return m(i), m(i + 1), b(j), b(j + 1)


def _as_points(points):
    """Return (pointer, n, keepalive, is_cuda) for int32 [n, 2] points (torch tensor or numpy)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(points, torch.Tensor):
        t = points
        if t.dtype != torch.int32:
            t = t.to(torch.int32)
        t = t.reshape(-1, 2).contiguous()
        return t.data_ptr(), t.shape[0], t, t.is_cuda
    a = np.ascontiguousarray(np.asarray(points, dtype=np.int32).reshape(-1, 2))
    return a.ctypes.data, a.shape[0], a, False


class Group:
    """In-process collective group of `world` ranks (include/hht.h hht_group_create): W contexts
    driven from W host threads run the multi-rank path with host-staged allreduces (tests)."""

    def __init__(self, world: int):
        self._lib = load()
        self._g = C.c_void_p()
        st = self._lib.hht_group_create(C.byref(self._g), world)
        if st:
            raise HHTError(st, "hht_group_create failed")
        self.world = world

    def close(self):
        if self._g:
            self._lib.hht_group_destroy(self._g)
            self._g = None


class HHT:
    """One libhht context (one device, one rank)."""

    def __init__(self, device: int = 0, halves: int = ALPHA | BETA, record_levels: bool = True,
                 force_int64: bool = False, profile: bool = False, mem_budget: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, tail_depth: int = 0,
                 prefetch: int = 0, variant: int = 0, group: Optional["Group"] = None, latency_path: int = 0,
                 stream: Optional[int] = None, tail_units: int = 0):
        self._lib = load()
        o = Opts()
        self._lib.hht_default_opts(C.byref(o))
        o.device, o.rank, o.world, o.halves = device, rank, world, halves
        o.record_levels, o.force_int64, o.profile = int(record_levels), int(force_int64), int(profile)
        o.mem_budget = mem_budget
        o.tail_depth = tail_depth
        o.prefetch = prefetch
        o.latency_path = latency_path
        o.variant = variant
        o.tail_units = tail_units
        if stream is not None:            # borrowed cudaStream_t handle (int), e.g. torch.cuda.Stream.cuda_stream
            o.stream = stream if stream else 1
        self._id = None
        if group is not None:
            o.group = group._g
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = C.cast(self._id, C.c_void_p)
        self._ctx = C.c_void_p()
        self._sink = None
        st = self._lib.hht_create(C.byref(self._ctx), C.byref(o))
        if st:
            raise HHTError(st, "hht_create failed")
        self.halves = halves
        self.world = world

    def _check(self, st: int):
        if st:
            raise HHTError(st, self._lib.hht_last_error(self._ctx).decode())

    def _order_after(self, t):
        """Device input: enqueue the library's work on torch's current stream of the tensor's device
        (hht_set_stream, borrowed), so the kernels or copies that produced `t` are ordered before the
        detection without a host synchronisation. Host input needs nothing (the library stages it)."""
        import torch
        if isinstance(t, torch.Tensor) and t.is_cuda:
            s = torch.cuda.current_stream(t.device).cuda_stream
            self._check(self._lib.hht_set_stream(self._ctx, C.c_void_p(s if s else 1)))   # 1: cudaStreamLegacy

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.hht_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # --- compute -----------------------------------------------------------------------------
    def detect(self, points, N: int, depth: int, threshold: int) -> "HHT":
        ptr, n, keep, _ = _as_points(points)
        self._order_after(keep)
        self._check(self._lib.hht_detect(self._ctx, C.c_void_p(ptr), n, N, depth, threshold))
        del keep
        return self

    def detect_batch(self, points, offsets: Sequence[int], N: int, depth: int, threshold: int) -> "HHT":
        ptr, n, keep, _ = _as_points(points)
        self._order_after(keep)
        offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        B = offs.shape[0] - 1
        self._check(self._lib.hht_detect_batch(self._ctx, C.c_void_p(ptr), offs.ctypes.data, B, N, depth,
                                               threshold))
        del keep
        return self

    # --- results -------------------------------------------------------------------------------
    def leaves_into(self, out: np.ndarray) -> int:
        """Copy every image's leaves as uint32 rows (image, half, i, j, votes) into `out` (a C-contiguous
        uint32 [cap, 5] array, e.g. a pinned buffer); returns the count."""
        assert out.dtype == np.uint32 and out.ndim == 2 and out.shape[1] == 5 and out.flags.c_contiguous
        cnt = C.c_int64(0)
        self._check(self._lib.hht_result_leaves(self._ctx, -1, C.c_void_p(out.ctypes.data), out.shape[0],
                                                C.byref(cnt)))
        return cnt.value

    def detect_trees(self, points, tree_offsets, N: int, depth: int, threshold: int):
        """Per-tree point sets: tree t (image t // H, half t % H in ALPHA, BETA order) gets
        points[tree_offsets[t]:tree_offsets[t+1]]."""
        ptr, n, keep, _ = _as_points(points)
        self._order_after(keep)
        to = np.ascontiguousarray(np.asarray(tree_offsets, dtype=np.int64))
        H = bin(self.halves).count("1")
        assert to.ndim == 1 and (to.shape[0] - 1) % H == 0 and to[-1] == n
        B = (to.shape[0] - 1) // H
        self._check(self._lib.hht_detect_trees(self._ctx, C.c_void_p(ptr), to.ctypes.data, B, N, depth, threshold))
        del keep
        return self

    def detect_image(self, img, mag_threshold: int, depth: int, threshold: int):
        """Sobel edge front end + detection of one square uint8 image [N, N] (row 0 = top), numpy or a
        CUDA tensor."""
        if hasattr(img, "data_ptr"):
            assert img.dtype.itemsize == 1 and img.is_contiguous() and img.dim() == 2
            N, ptr, keep = int(img.shape[0]), img.data_ptr(), img
            assert img.shape[1] == N
            self._order_after(img)          # the producer of a device image is ordered first
        else:
            keep = np.ascontiguousarray(img, dtype=np.uint8)
            assert keep.ndim == 2 and keep.shape[0] == keep.shape[1]
            N, ptr = keep.shape[0], keep.ctypes.data
        self._check(self._lib.hht_detect_image(self._ctx, C.c_void_p(ptr), N, mag_threshold, depth, threshold))
        del keep

    def lines(self, image: int = -1) -> np.ndarray:
        """int64 [k, 5] (image, half, i, j, live votes): solution() with point removal
        over the last detect's candidate leaves, depth-first order per tree."""
        cnt = C.c_int64(0)
        self._check(self._lib.hht_result_lines(self._ctx, image, None, 0, C.byref(cnt)))
        out = (Leaf * max(cnt.value, 1))()
        self._check(self._lib.hht_result_lines(self._ctx, image, out, cnt.value, C.byref(cnt)))
        return np.frombuffer(out, dtype=np.uint32, count=5 * cnt.value).reshape(-1, 5).astype(np.int64)

    def line_points(self, image: int = -1) -> np.ndarray:
        """int64 [k, 2] (line, point): the points each removal-on line emitted (hht_result_line_points),
        sorted by line then point; line indexes lines(image)."""
        cnt = C.c_int64(0)
        self._check(self._lib.hht_result_line_points(self._ctx, image, None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), dtype=np.uint32)
        self._check(self._lib.hht_result_line_points(self._ctx, image, out.ctypes.data, cnt.value, C.byref(cnt)))
        return out[:cnt.value].astype(np.int64)

    def edges(self):
        """(alpha, beta) int32 [k, 2] (x, y) edge points of the last detect_image, raster order."""
        na, nb = C.c_int64(0), C.c_int64(0)
        self._check(self._lib.hht_result_edges(self._ctx, None, 0, C.byref(na), C.byref(nb)))
        out = np.empty((max(na.value + nb.value, 1), 2), dtype=np.int32)
        self._check(self._lib.hht_result_edges(self._ctx, out.ctypes.data, out.shape[0], C.byref(na),
                                               C.byref(nb)))
        return out[:na.value].copy(), out[na.value:na.value + nb.value].copy()

    def set_leaf_sink(self, out: Optional[np.ndarray]):
        """Stream every later detect's leaf rows (image, half, i, j, votes) into `out` (a C-contiguous
        uint32 [cap, 5] array, ideally pinned) while the detection runs; None removes the sink."""
        if out is None:
            self._check(self._lib.hht_set_leaf_sink(self._ctx, None, 0))
            self._sink = None
            return
        assert out.dtype == np.uint32 and out.ndim == 2 and out.shape[1] == 5 and out.flags.c_contiguous
        self._sink = out
        self._check(self._lib.hht_set_leaf_sink(self._ctx, C.c_void_p(out.ctypes.data), out.shape[0]))

    def set_leaf_sink_packed(self, out: Optional[np.ndarray]):
        """Stream every later detect's leaf rows as packed uint64 (i << 48 | j << 32 | votes) into
        `out` (a C-contiguous uint64 [cap] array, ideally pinned); None removes the sink. The tree of
        each row follows from tree_offsets(). Needs depth <= 16."""
        if out is None:
            self._check(self._lib.hht_set_leaf_sink_packed(self._ctx, None, 0))
            self._sink = None
            return
        assert out.dtype == np.uint64 and out.ndim == 1 and out.flags.c_contiguous
        self._sink = out
        self._check(self._lib.hht_set_leaf_sink_packed(self._ctx, C.c_void_p(out.ctypes.data), out.shape[0]))

    def tree_offsets(self) -> np.ndarray:
        """uint64 [ntrees + 1]: index of each tree's first detected line in the leaf order of the last
        detect (tree t = image t / H, half index t % H, ALPHA first)."""
        nt = C.c_int64()
        self._check(self._lib.hht_result_tree_offsets(self._ctx, None, 0, C.byref(nt)))
        out = np.zeros(nt.value + 1, dtype=np.uint64)
        self._check(self._lib.hht_result_tree_offsets(self._ctx, C.c_void_p(out.ctypes.data), out.shape[0], C.byref(nt)))
        return out

    def leaves(self, image: int = -1) -> np.ndarray:
        """int64 [L, 5]: (image, half, i, j, votes) in image, half, depth-first order."""
        if image == -1:
            cnt = C.c_int64(0)
            st = self._lib.hht_result_leaves(self._ctx, -1, None, 0, C.byref(cnt))
            if st and cnt.value == 0:
                self._check(st)
            buf = np.empty((max(cnt.value, 1), 5), dtype=np.uint32)
            n = self.leaves_into(buf)
            return buf[:n].astype(np.int64)
        cnt = C.c_int64(0)
        st = self._lib.hht_result_leaves(self._ctx, image, None, 0, C.byref(cnt))
        if st and cnt.value == 0:
            self._check(st)
        out = (Leaf * max(cnt.value, 1))()
        self._check(self._lib.hht_result_leaves(self._ctx, image, out, cnt.value, C.byref(cnt)))
        arr = np.frombuffer(out, dtype=np.uint32, count=5 * cnt.value).reshape(-1, 5).astype(np.int64)
        return arr

    def level(self, image: int, half: int, level: int) -> np.ndarray:
        """uint32 [k, 3]: (a, c, votes) of the visited regions of one tree at one level."""
        cnt = C.c_int64(0)
        st = self._lib.hht_result_level(self._ctx, image, half, level, None, 0, C.byref(cnt))
        if st and cnt.value == 0:
            self._check(st)
        out = np.zeros((max(cnt.value, 1), 3), dtype=np.uint32)
        self._check(self._lib.hht_result_level(self._ctx, image, half, level, out.ctypes.data, cnt.value,
                                               C.byref(cnt)))
        return out[:cnt.value]

    def stats(self) -> dict:
        s = Stats()
        self._check(self._lib.hht_result_stats(self._ctx, C.byref(s)))
        L = s.levels
        return {"tests": s.tests, "votes": s.votes, "leaves": s.leaves, "pairs": s.pairs,
                "visited": list(s.visited)[:L], "split": list(s.split)[:L], "h2d_bytes": s.h2d_bytes,
                "d2h_bytes": s.d2h_bytes, "levels": L, "int_bits": s.int_bits, "ranges": s.ranges,
                "images": s.images, "ms": s.ms, "leaves_streamed": s.leaves_streamed,
                "latency_path": s.latency_path}

    def profile(self) -> dict:
        p = Profile()
        self._check(self._lib.hht_result_profile(self._ctx, C.byref(p)))
        return {name: {"launches": p.launches[k], "ms": p.ms[k], "bytes": p.bytes[k], "ops": p.ops[k]}
                for k, name in enumerate(PROFILE_CLASSES)}

    def launches(self) -> list:
        """Per-launch log of the last detect (profile=True): [(class name, algorithmic bytes, ms)]."""
        cnt = C.c_int64(0)
        st = self._lib.hht_result_launches(self._ctx, None, 0, C.byref(cnt))
        if st and cnt.value == 0:
            self._check(st)
        out = (Launch * max(cnt.value, 1))()
        self._check(self._lib.hht_result_launches(self._ctx, out, cnt.value, C.byref(cnt)))
        return [(PROFILE_CLASSES[out[i].cls], out[i].bytes, out[i].ms) for i in range(cnt.value)]

    def timer_begin(self):
        self._check(self._lib.hht_timer_begin(self._ctx))

    def timer_end(self) -> float:
        ms = C.c_double(0)
        self._check(self._lib.hht_timer_end(self._ctx, C.byref(ms)))
        return ms.value
