"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/hht_oracle.c header): the paper's edge front end,
written out plainly with numpy for the tests of the GPU front end. Never imported by the product.

PAPER.md:67 (§3): "Sobel's gradient operator is being applied" to the grayscale image, and the edge
points are split into two sets: "One called ALPHA with edge points belonging to lines" whose slope
magnitude is at most 1 (§1, "absolute value of slope less than or equal to 1"), the other
(BETA) handled by "reversing the roles of co-ordinates". The paper fixes neither the kernels, the
magnitude, the threshold nor the axis convention; the readings (R18-R21) follow SPEC.md's
DESIGN DECISIONS:
  * gx = [[-1,0,1],[-2,0,2],[-1,0,1]], gy = [[-1,-2,-1],[0,0,0],[1,2,1]] in geometric coordinates:
    x = column, y = H-1-row (y grows upwards), so gy = sum_dx w(dx) (I(x+dx, y+1) - I(x+dx, y-1))
    with w = (1, 2, 1), and gx = sum_dy w(dy) (I(x+1, y+dy) - I(x-1, y+dy));
  * border pixels get gradient (0, 0); magnitude |gx| + |gy| (L1, no square roots);
  * a pixel is an edge point iff |gx| + |gy| >= thr and thr > 0;
  * ALPHA iff |gx| <= |gy| (tie to ALPHA: the slope bound is inclusive), else BETA;
  * each set in original raster order: row 0 (top) first, columns ascending within a row.
"""
from __future__ import annotations

import numpy as np

W3 = (1, 2, 1)


def sobel(img: np.ndarray):
    """img: uint8 [H, W], row 0 = top. Returns int32 (gx, gy) [H, W] in geometric orientation."""
    img = np.asarray(img)
    if img.ndim != 2 or img.shape[0] < 3 or img.shape[1] < 3:
        raise ValueError("sobel needs an image of at least 3x3 pixels")
    H, Wd = img.shape
    I = img.astype(np.int32)
    gx = np.zeros((H, Wd), np.int32)
    gy = np.zeros((H, Wd), np.int32)
    for r in range(1, H - 1):
        for c in range(1, Wd - 1):
            sx = sy = 0
            for k, d in enumerate((-1, 0, 1)):
                # geometric y+d is row r-d (rows count downwards)
                sx += W3[k] * (int(I[r - d, c + 1]) - int(I[r - d, c - 1]))
                sy += W3[k] * (int(I[r - 1, c + d]) - int(I[r + 1, c + d]))
            gx[r, c] = sx
            gy[r, c] = sy
    return gx, gy


def partition_edges(gx: np.ndarray, gy: np.ndarray, thr: int):
    """(alpha, beta): int32 [k, 2] (x, y) edge points of each set, original raster order."""
    H, Wd = gx.shape
    alpha, beta = [], []
    if thr > 0:
        for r in range(H):
            for c in range(Wd):
                ax, ay = abs(int(gx[r, c])), abs(int(gy[r, c]))
                if ax + ay >= thr:
                    (alpha if ax <= ay else beta).append((c, H - 1 - r))
    a = np.array(alpha, np.int32).reshape(-1, 2)
    b = np.array(beta, np.int32).reshape(-1, 2)
    return a, b


def edges(img: np.ndarray, thr: int):
    gx, gy = sobel(img)
    return partition_edges(gx, gy, thr)
