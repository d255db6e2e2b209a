"""ctypes wrapper around oracle/hht_oracle.c -- ORACLE, TEST INFRASTRUCTURE ONLY.

Argument marshalling only; every step of the method is in the C file, which cites the paper.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
import threading
from typing import Dict, Tuple

import numpy as np

ALPHA = 1
BETA = 2
MAXLEV = 64

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hht_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/hht_oracle.c with gcc (plain -O2, no OpenMP, no vector intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            i32, i64, p = C.c_int32, C.c_int64, C.c_void_p
            lib.oracle_corner_below.argtypes = [i64, i64, i32, i32, i64, i64]
            lib.oracle_corner_below.restype = C.c_int
            lib.oracle_code.argtypes = [i32, i32, i32, i32, i32, i32, i64, i64]
            lib.oracle_code.restype = C.c_int
            lib.oracle_generic_code.argtypes = [i64] * 7
            lib.oracle_generic_code.restype = C.c_int
            lib.oracle_circle_passes.argtypes = [i32, i32, i32, i32, i32, i32, i64, i64]
            lib.oracle_circle_passes.restype = C.c_int
            lib.oracle_circle_mb_passes.argtypes = [i32, i32, i32, i32, i32, i32, i64, i64]
            lib.oracle_circle_mb_passes.restype = C.c_int
            lib.oracle_region_votes.argtypes = [p, i64, i32, i32, i32, i32, i64, i64, i32]
            lib.oracle_region_votes.restype = i64
            lib.oracle_dense_votes.argtypes = [p, i64, i32, i32, i32, i32, p]
            lib.oracle_dense_votes.restype = None
            lib.oracle_detect.argtypes = [p, i64, i32, i32, i64, i32, i32, i64]
            lib.oracle_detect.restype = p
            lib.oracle_detect_removal.argtypes = [p, i64, i32, i32, i64, i32]
            lib.oracle_detect_removal.restype = p
            lib.oracle_result_support_count.argtypes = [p]
            lib.oracle_result_support_count.restype = i64
            lib.oracle_result_support.argtypes = [p, p]
            lib.oracle_result_support.restype = None
            lib.oracle_detect_subtree.argtypes = [p, i64, i32, i32, i64, i32, i32, i64, i64]
            lib.oracle_detect_subtree.restype = p
            lib.oracle_result_level_count.argtypes = [p, i32, i32]
            lib.oracle_result_level_count.restype = i64
            lib.oracle_result_level.argtypes = [p, i32, i32, p]
            lib.oracle_result_level.restype = None
            lib.oracle_result_leaf_count.argtypes = [p]
            lib.oracle_result_leaf_count.restype = i64
            lib.oracle_result_leaves.argtypes = [p, p]
            lib.oracle_result_leaves.restype = None
            lib.oracle_result_stats.argtypes = [p, p]
            lib.oracle_result_stats.restype = None
            lib.oracle_result_free.argtypes = [p]
            lib.oracle_result_free.restype = None
            _lib = lib
    return _lib


def _pts(points) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(points, dtype=np.int32).reshape(-1, 2))
    return a


def corner_below(ex: int, ey: int, N: int, D: int, i: int, j: int) -> int:
    return _load().oracle_corner_below(ex, ey, N, D, i, j)


def code(x: int, y: int, half: int, N: int, D: int, level: int, a: int, c: int) -> int:
    return _load().oracle_code(x, y, half, N, D, level, a, c)


def generic_code(m_num: int, m_den: int, b_num: int, b_den: int, x0: int, y0: int, side: int) -> int:
    return _load().oracle_generic_code(m_num, m_den, b_num, b_den, x0, y0, side)


def circle_passes(x: int, y: int, half: int, N: int, D: int, level: int, a: int, c: int) -> int:
    return _load().oracle_circle_passes(x, y, half, N, D, level, a, c)


def circle_mb_passes(x: int, y: int, half: int, N: int, D: int, level: int, a: int, c: int) -> int:
    return _load().oracle_circle_mb_passes(x, y, half, N, D, level, a, c)


def region_votes(points, half: int, N: int, D: int, level: int, a: int, c: int, variant: int = 0) -> int:
    p = _pts(points)
    return int(_load().oracle_region_votes(p.ctypes.data, p.shape[0], half, N, D, level, a, c, variant))


def dense_votes(points, half: int, N: int, D: int, level: int) -> np.ndarray:
    """acc[c, a] = votes of level-`level` region (a, c) over all points."""
    p = _pts(points)
    side = 1 << level
    acc = np.zeros((side, side), dtype=np.uint32)
    _load().oracle_dense_votes(p.ctypes.data, p.shape[0], half, N, D, level, acc.ctypes.data)
    return acc


@dataclasses.dataclass
class OracleResult:
    N: int
    D: int
    T: int
    halves: int
    levels: Dict[Tuple[int, int], np.ndarray]   # (half, level) -> uint32 [k, 3] (a, c, votes), DFS order
    leaves: np.ndarray                           # uint32 [L, 4] (half, i, j, votes), DFS order
    tests: int
    votes: int
    truncated: bool
    visited: Dict[int, np.ndarray]               # half -> int64 [MAXLEV]
    split: Dict[int, np.ndarray]


def _collect(lib, h, N, D, T, halves) -> OracleResult:
    try:
        st = np.zeros(8 + 4 * MAXLEV, dtype=np.int64)
        lib.oracle_result_stats(h, st.ctypes.data)
        if st[4]:
            raise MemoryError("oracle ran out of memory")
        levels = {}
        for half in (ALPHA, BETA):
            if not (halves & half):
                continue
            for lev in range(D + 1):
                n = lib.oracle_result_level_count(h, half, lev)
                arr = np.zeros((n, 3), dtype=np.uint32)
                if n:
                    lib.oracle_result_level(h, half, lev, arr.ctypes.data)
                levels[(half, lev)] = arr
        nl = lib.oracle_result_leaf_count(h)
        leaves = np.zeros((nl, 4), dtype=np.uint32)
        if nl:
            lib.oracle_result_leaves(h, leaves.ctypes.data)
        hi = {ALPHA: 0, BETA: 1}
        visited = {hf: st[8 + hi[hf] * MAXLEV: 8 + (hi[hf] + 1) * MAXLEV].copy() for hf in (ALPHA, BETA)}
        split = {hf: st[8 + (2 + hi[hf]) * MAXLEV: 8 + (3 + hi[hf]) * MAXLEV].copy() for hf in (ALPHA, BETA)}
        return OracleResult(N, D, T, halves, levels, leaves, int(st[0]), int(st[1]), bool(st[3]),
                            visited, split)
    finally:
        lib.oracle_result_free(h)


def detect(points, N: int, D: int, T: int, halves: int = ALPHA | BETA, variant: int = 0,
           max_tests: int = 0) -> OracleResult:
    """Recursive DFS detector (removal off). variant 0 = exact 4-bit code,
    1 = FHT circumcircle test in lattice units (square regions), 2 = FHT circumcircle test in
    (m, b) units (2s/2^D x 3Ns/2^D rectangles; reading R22). max_tests > 0 stops the walk once that many code evaluations were
    done (bounded CPU-baseline samples; result.truncated is then True)."""
    p = _pts(points)
    lib = _load()
    h = lib.oracle_detect(p.ctypes.data, p.shape[0], N, D, T, halves, variant, max_tests)
    if not h:
        raise ValueError("oracle_detect rejected its arguments")
    return _collect(lib, h, N, D, T, halves)


def detect_removal(points, N: int, D: int, T: int, halves: int = ALPHA | BETA):
    """The detector with solution()'s point removal ON: returns (lines, support)
    where lines is uint32 [k, 4] (half, i, j, live votes) in emission (depth-first) order and support
    is uint32 [m, 2] (line index, point index): the points each line emitted and removed."""
    p = _pts(points)
    lib = _load()
    h = lib.oracle_detect_removal(p.ctypes.data, p.shape[0], N, D, T, halves)
    if not h:
        raise ValueError("oracle_detect_removal rejected its arguments")
    try:
        nl = lib.oracle_result_leaf_count(h)
        lines = np.zeros((nl, 4), dtype=np.uint32)
        if nl:
            lib.oracle_result_leaves(h, lines.ctypes.data)
        ns = lib.oracle_result_support_count(h)
        sup = np.zeros((ns, 2), dtype=np.uint32)
        if ns:
            lib.oracle_result_support(h, sup.ctypes.data)
        return lines, sup
    finally:
        lib.oracle_result_free(h)


def detect_subtree(points, N: int, D: int, T: int, half: int, level: int, a: int, c: int) -> OracleResult:
    p = _pts(points)
    lib = _load()
    h = lib.oracle_detect_subtree(p.ctypes.data, p.shape[0], N, D, T, half, level, a, c)
    if not h:
        raise MemoryError("oracle_detect_subtree")
    return _collect(lib, h, N, D, T, half)
