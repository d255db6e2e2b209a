"""Seeded synthetic edge-point generator (shared input module).

This module is the ONE piece of code both sides consume: the CPU oracle (``oracle/``, tests only)
and the CUDA path (``libhht.so`` via ``paper_1007_0547_b200.hht``). It holds none of the method's
arithmetic -- no corner signs, codes, votes or region geometry -- it only draws integer points.

Recipe (SURVEY.md §8(d) "Generator", readings listed in DESIGN.md §3):

* PRNG: counter-based splitmix64. A stream is keyed by (config id, image index, purpose); value k
  of a stream is ``mix(key + (k+1)*GAMMA)``. Uniform integers in [0, K) use the high-32-bit
  multiply ``((r >> 32) * K) >> 32`` (bias <= K/2^32; deterministic, vectorisable).
* Line (k points, jitter J): slope m = A/2^16, A uniform in [-2^16, 2^16] (|m| <= 1);
  intercept b = Q/2^16, Q uniform in [-N*2^16, 2N*2^16) (b in [-N, 2N), BASELINE.json configs[0]).
  Dependent coordinate u(t) = floor((A*t + Q + 2^15) / 2^16) (round half up). Valid t are those
  with J <= u(t) <= N-1-J; fewer than k valid -> redraw the line. k distinct t are the first k of
  the valid t ordered by fresh random keys; each emits u(t)+delta, delta uniform in [-J, J].
  An ALPHA line emits (t, u+delta); a BETA line emits (u+delta, t) ("reversing the
  roles of co-ordinates"). A line's half is ALPHA when the config is ALPHA-only, else a fair coin.
* Noise: independent uniform (x, y) in [0, N)^2; duplicates kept (a multiset, A15).
* Order: line points, then noise, then one seeded permutation of the whole array (argsort of
  random keys), so contiguous sharding across ranks is balanced.

All five BASELINE.json configs are in ``CONFIGS``; ``scene()`` builds arbitrary small scenes for
tests.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np

ALPHA = 1
BETA = 2

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def _mix_int(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_key(*parts: int) -> int:
    """Derive a 64-bit stream key from integer parts (config id, image, purpose, ...)."""
    k = 0x243F6A8885A308D3
    for p in parts:
        k = _mix_int(k ^ _mix_int((int(p) + _GAMMA) & _M64))
    return k


class Stream:
    """Counter-based splitmix64 stream: value k is mix(key + (k+1)*GAMMA)."""

    def __init__(self, key: int):
        self.key = int(key) & _M64
        self.pos = 0

    def u64(self, n: int) -> np.ndarray:
        idx = np.arange(self.pos + 1, self.pos + 1 + n, dtype=np.uint64)
        self.pos += n
        with np.errstate(over="ignore"):
            z = np.uint64(self.key) + idx * np.uint64(_GAMMA)
            return _mix_np(z)

    def below(self, k: int, n: int) -> np.ndarray:
        """n uniform integers in [0, k), k < 2^32, as int64."""
        assert 0 < k < (1 << 32)
        r = self.u64(n) >> np.uint64(32)
        with np.errstate(over="ignore"):
            return ((r * np.uint64(k)) >> np.uint64(32)).astype(np.int64)

    def uniform(self, lo: int, hi: int, n: int) -> np.ndarray:
        """n uniform integers in the closed range [lo, hi]."""
        return self.below(hi - lo + 1, n) + lo


@dataclasses.dataclass(frozen=True)
class LineTruth:
    half: int      # ALPHA or BETA
    A: int         # slope numerator, m = A / 2^16
    Q: int         # intercept numerator, b = Q / 2^16
    k: int         # points emitted


@dataclasses.dataclass(frozen=True)
class Config:
    cid: int
    N: int
    D: int
    T: int
    halves: int        # bitmask ALPHA|BETA
    images: int
    lines: int
    per_line: int
    jitter: int
    noise: int
    text: str

    @property
    def alpha_only(self) -> bool:
        return self.halves == ALPHA


# BASELINE.json configs[0..4] -> ids 1..5 (readings in DESIGN.md §3).
CONFIGS = {
    1: Config(1, 64, 6, 20, ALPHA, 1, 3, 40, 0, 100, "64x64, 3x40 + 100 noise, ALPHA only, D=6, T=20"),
    2: Config(2, 512, 9, 50, ALPHA | BETA, 1, 20, 200, 1, 13107,
              "512x512, 20x200 +-1px + 5% noise (13107), both halves, D=9, T=50"),
    3: Config(3, 2048, 11, 200, ALPHA | BETA, 1, 100, 1000, 1, 300000,
              "2048x2048, 100x1000 +-1px + 300k noise, both halves, D=11, T=200"),
    4: Config(4, 1024, 10, 100, ALPHA | BETA, 256, 50, 500, 0, 25000,
              "256 x 1024x1024, 50x500 + 25k noise each, both halves, D=10, T=100"),
    5: Config(5, 8192, 13, 1000, ALPHA | BETA, 1, 1000, 4000, 2, 12000000,
              "8192x8192, 1000x4000 +-2px + 12M noise (16M points), both halves, D=13, T=1000"),
}

P_LINES, P_NOISE, P_SHUFFLE = 1, 2, 3


def _draw_line(rng: Stream, N: int, k: int, J: int, alpha_only: bool):
    while True:
        A = int(rng.uniform(-(1 << 16), 1 << 16, 1)[0])
        Q = int(rng.uniform(-N * (1 << 16), 2 * N * (1 << 16) - 1, 1)[0])
        t = np.arange(N, dtype=np.int64)
        u = (A * t + Q + (1 << 15)) // (1 << 16)          # floor division (numpy floors negatives)
        ok = (u >= J) & (u <= N - 1 - J)
        vt = t[ok]
        if vt.size < k:
            continue
        keys = rng.u64(vt.size)
        chosen = vt[np.argsort(keys, kind="stable")[:k]]
        uu = (A * chosen + Q + (1 << 15)) // (1 << 16)
        delta = rng.uniform(-J, J, k) if J > 0 else np.zeros(k, dtype=np.int64)
        half = ALPHA if alpha_only else (ALPHA if int(rng.below(2, 1)[0]) == 0 else BETA)
        dep = uu + delta
        if half == ALPHA:
            pts = np.stack([chosen, dep], axis=1)
        else:
            pts = np.stack([dep, chosen], axis=1)
        return pts, LineTruth(half, A, Q, k)


def scene(N: int, n_lines: int, per_line: int, jitter: int, n_noise: int, alpha_only: bool,
          *key_parts: int) -> Tuple[np.ndarray, List[LineTruth]]:
    """Generate one image's edge points: int32 [E, 2] (x, y), C-contiguous, plus line truth."""
    assert N >= 1 and per_line <= N and 2 * jitter < N
    rng_l = Stream(stream_key(*key_parts, P_LINES))
    chunks, truth = [], []
    for _ in range(n_lines):
        p, tr = _draw_line(rng_l, N, per_line, jitter, alpha_only)
        chunks.append(p)
        truth.append(tr)
    if n_noise:
        rng_n = Stream(stream_key(*key_parts, P_NOISE))
        xy = rng_n.below(N, 2 * n_noise).reshape(n_noise, 2)
        chunks.append(xy)
    pts = np.concatenate(chunks, axis=0) if chunks else np.zeros((0, 2), dtype=np.int64)
    if pts.shape[0] > 1:
        rng_s = Stream(stream_key(*key_parts, P_SHUFFLE))
        pts = pts[np.argsort(rng_s.u64(pts.shape[0]), kind="stable")]
    out = np.ascontiguousarray(pts, dtype=np.int32)
    assert out.size == 0 or (out.min() >= 0 and out.max() < N)
    return out, truth


def config_image(cid: int, image: int = 0) -> Tuple[np.ndarray, List[LineTruth]]:
    c = CONFIGS[cid]
    return scene(c.N, c.lines, c.per_line, c.jitter, c.noise, c.alpha_only, cid, image)


def config_batch(cid: int, images: int | None = None) -> Tuple[np.ndarray, np.ndarray]:
    """All images of a config concatenated: points int32 [sum E, 2] and offsets int64 [B+1]."""
    c = CONFIGS[cid]
    B = c.images if images is None else images
    parts = [config_image(cid, b)[0] for b in range(B)]
    offs = np.zeros(B + 1, dtype=np.int64)
    offs[1:] = np.cumsum([p.shape[0] for p in parts])
    return np.ascontiguousarray(np.concatenate(parts, axis=0)), offs


def random_scene(seed: int, N: int, max_lines: int = 3, max_noise: int = 60,
                 alpha_only: bool = False) -> np.ndarray:
    """Small random scene for property tests: line count, length, jitter, noise all drawn."""
    r = Stream(stream_key(0xC0FFEE, seed))
    nl = int(r.below(max_lines + 1, 1)[0])
    per = int(r.uniform(1, max(1, N // 2), 1)[0])
    J = int(r.below(2, 1)[0]) if N > 4 else 0
    nn = int(r.below(max_noise + 1, 1)[0])
    pts, _ = scene(N, nl, per, J, nn, alpha_only, 0xC0FFEE, seed, 7)
    return pts


def shard(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced shard [lo, hi) of n items for rank in a world of ``world`` ranks."""
    assert 0 <= rank < world
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
