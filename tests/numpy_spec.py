"""A second, independent restatement of the frozen pixel spec (
SURVEY §8 A1/A2), written with numpy array operations instead of the C
oracle's loops -- TEST INFRASTRUCTURE ONLY.  The pixel stages have no
reference implementation, so the C oracle (oracle/tangram_oracle.c) is the
checker; this module cross-checks the oracle itself, so a misreading of the
spec shared by the oracle and the kernels would have to be made a third
time, in a different style, to go unnoticed.

* mask: fg0 = max_c |cur - prev| > T, then a (2r+1)^2 square dilation as the
  OR of shifted copies of the zero-padded mask (outside = background);
* cells: 16 x 16 blocks by reshape; popcount by sum; the fg bounding box
  inside each block by any() along each axis; packed as count | x0 << 9 |
  x1 << 13 | y0 << 17 | y1 << 21, 0 for empty cells;
* RoIs: 8-connected components of active cells by breadth-first search,
  ordered by their first cell in raster order, each boxed by the min / max
  of its cells' pixel extents.
"""
from __future__ import annotations

from collections import deque

import numpy as np

CELL = 16


def mask(cur: np.ndarray, prev: np.ndarray, W: int, H: int, T: int, r: int) -> np.ndarray:
    """Dilated foreground, bool (H, W)."""
    c = cur[:H, :3 * W].reshape(H, W, 3).astype(np.int16)
    p = prev[:H, :3 * W].reshape(H, W, 3).astype(np.int16)
    fg0 = np.abs(c - p).max(axis=2) > T
    padded = np.pad(fg0, r)
    out = np.zeros_like(fg0)
    for dy in range(2 * r + 1):
        for dx in range(2 * r + 1):
            out |= padded[dy:dy + H, dx:dx + W]
    return out


def pack_bits(fg: np.ndarray) -> np.ndarray:
    """bool (H, W) -> the oracle's rows of ceil(W/32) little-endian words."""
    H, W = fg.shape
    nw = (W + 31) // 32
    padded = np.zeros((H, nw * 32), bool)
    padded[:, :W] = fg
    return np.packbits(padded, axis=1, bitorder="little").view(np.uint32)


def cells(fg: np.ndarray) -> np.ndarray:
    H, W = fg.shape
    cy, cx = -(-H // CELL), -(-W // CELL)
    padded = np.zeros((cy * CELL, cx * CELL), bool)
    padded[:H, :W] = fg
    blk = padded.reshape(cy, CELL, cx, CELL).transpose(0, 2, 1, 3)  # [cy, cx, y, x]
    count = blk.sum(axis=(2, 3)).astype(np.uint32)
    cols = blk.any(axis=2)  # [cy, cx, x]
    rows = blk.any(axis=3)  # [cy, cx, y]
    x0 = cols.argmax(axis=2)
    x1 = CELL - 1 - cols[..., ::-1].argmax(axis=2)
    y0 = rows.argmax(axis=2)
    y1 = CELL - 1 - rows[..., ::-1].argmax(axis=2)
    packed = count | (x0.astype(np.uint32) << 9) | (x1.astype(np.uint32) << 13) | \
        (y0.astype(np.uint32) << 17) | (y1.astype(np.uint32) << 21)
    return np.where(count > 0, packed, 0).astype(np.uint32)


def rois(cell_grid: np.ndarray) -> list[tuple[int, int, int, int]]:
    cy, cx = cell_grid.shape
    active = cell_grid != 0
    seen = np.zeros_like(active)
    out = []
    for sy, sx in zip(*np.nonzero(active)):  # raster order: row-major
        if seen[sy, sx]:
            continue
        seen[sy, sx] = True
        todo = deque([(sy, sx)])
        bx0 = by0 = 1 << 30
        bx1 = by1 = -1
        while todo:
            y, x = todo.popleft()
            v = int(cell_grid[y, x])
            bx0 = min(bx0, x * CELL + (v >> 9 & 15))
            bx1 = max(bx1, x * CELL + (v >> 13 & 15))
            by0 = min(by0, y * CELL + (v >> 17 & 15))
            by1 = max(by1, y * CELL + (v >> 21 & 15))
            for ny in (y - 1, y, y + 1):
                for nx in (x - 1, x, x + 1):
                    if 0 <= ny < cy and 0 <= nx < cx and active[ny, nx] and not seen[ny, nx]:
                        seen[ny, nx] = True
                        todo.append((ny, nx))
        out.append((bx0, by0, bx1 - bx0 + 1, by1 - by0 + 1))
    return out
