"""Rect algebra (geometry.hpp:28-68) and the C07 granularity property
(acceptance_test.cpp:310-347) -- the reference's own expectations.

Geometry KATs and the 64x64 pixel-grid oracle follow geometry_test.cpp:27-103
on the host mirror (api.area / overlap_area / contains / enclosing_rect, the
same arithmetic the device's rect_core.cuh runs).  C07 runs the oracle's
partition (the reference's own partition() when oracle/_ref is built); the
device partition gets the same check in test_gpu_parity.py.
"""
import math

import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A

R = A.Rect


def test_geometry_known_answers():
    assert A.area(R(0, 0, 3, 4)) == 12 and A.area(R(10, 20, 1, 1)) == 1 and A.area(R(0, 0, 0, 5)) == 0
    assert A.overlap_area(R(30, 10, 30, 20), R(0, 0, 50, 50)) == 400
    assert A.overlap_area(R(0, 0, 50, 50), R(30, 10, 30, 20)) == 400
    assert A.overlap_area(R(0, 0, 10, 10), R(10, 0, 10, 10)) == 0
    assert A.overlap_area(R(0, 0, 10, 10), R(20, 20, 5, 5)) == 0
    assert A.overlap_area(R(2, 2, 4, 4), R(0, 0, 50, 50)) == 16
    assert A.contains(R(0, 0, 10, 10), R(0, 0, 10, 10))
    assert A.contains(R(0, 0, 10, 10), R(2, 3, 4, 5))
    assert not A.contains(R(0, 0, 10, 10), R(5, 5, 6, 5))
    assert not A.contains(R(2, 2, 4, 4), R(0, 0, 10, 10))
    assert A.enclosing_rect([R(5, 5, 10, 10), R(30, 10, 30, 20)]) == R(5, 5, 55, 25)
    assert A.enclosing_rect([R(7, 9, 3, 2)]) == R(7, 9, 3, 2)
    with pytest.raises(A.InvalidArgument, match="empty rect set"):
        A.enclosing_rect([])


def test_geometry_pixel_grid_oracle():
    rng = O.Rng(O.derive_seed(99, "geometry-oracle"))

    def random_rect():
        w = rng.uniform_int(1, 32)
        h = rng.uniform_int(1, 32)
        return R(rng.uniform_int(0, 64 - w), rng.uniform_int(0, 64 - h), w, h)

    for _ in range(500):
        a, b = random_rect(), random_rect()
        px = sum(1 for y in range(max(a.y, b.y), min(a.top(), b.top()))
                 for x in range(max(a.x, b.x), min(a.right(), b.right())))
        assert A.overlap_area(a, b) == px
        enc = A.enclosing_rect([a, b])
        assert A.contains(enc, a) and A.contains(enc, b)
        x0, y0 = min(a.x, b.x), min(a.y, b.y)
        assert enc == R(x0, y0, max(a.right(), b.right()) - x0, max(a.top(), b.top()) - y0)


def c07_means(partition_bytes, n_scenes=10):
    """acceptance_test.cpp:310-347: mean bytes per scene for grids 2/4/6 and
    for whole frames."""
    mean_full, by_grid = 0.0, {2: 0.0, 4: 0.0, 6: 0.0}
    for s in range(1, n_scenes + 1):
        cfg = O.gen_cfg(n_frames=120, seed=s)
        t_us, frames = O.generate_trace(cfg)
        full = 0.0
        for rois in frames:
            if rois:
                full += math.ceil(cfg.frame_width * cfg.frame_height * 1.5)
        mean_full += full / n_scenes
        for z in (2, 4, 6):
            b = 0.0
            for i, rois in enumerate(frames):
                b += partition_bytes(i, cfg.frame_width, cfg.frame_height, t_us[i], z, rois)
            by_grid[z] += b / n_scenes
    return mean_full, by_grid


def check_c07(mean_full, by_grid):
    slack = 1.02  # enclosing-rectangle tie allowance (acceptance_test.cpp:342)
    assert by_grid[6] <= by_grid[4] * slack
    assert by_grid[4] <= by_grid[2] * slack
    assert by_grid[2] <= mean_full * slack
    assert by_grid[6] > 0.0


@pytest.mark.parametrize("lib", ["port", "ref"])
def test_c07_finer_grids_transmit_no_more_bytes(lib):
    if lib == "ref" and not O.have_ref():
        pytest.skip("oracle/_ref absent")

    def pb(i, W, H, t, z, rois):
        return float(sum(p["size_bytes"] for p in
                         O.partition(i, W, H, t, 1_000_000, z, z, rois, 1.5, 0, lib=lib)))

    check_c07(*c07_means(pb))
