"""The frozen pixel spec (A1 mask, A2 cells + RoIs) pinned by two
independent restatements: the C oracle (oracle/tangram_oracle.c, the
checker the GPU parity tests use) must equal tests/numpy_spec.py, written
with numpy array operations, on generator frames and on adversarial random
frames, for several dilation radii and thresholds.  Also: the region
synthesizer the full-size canvas checks use equals crops of whole frames."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import numpy_spec as S


def _pair(W, H, seed, roi_max_dim=400, t=3):
    cfg = O.gen_cfg(seed=seed, n_frames=t + 1, fps=30.0, frame_width=W, frame_height=H,
                    roi_max_dim=roi_max_dim, roi_proportion_mean=0.2)
    _, rects = O.generate_trace(cfg)
    ps = O.derive_seed(seed, "pixels")
    return O.synth_frame(W, H, ps, t, rects[t]), O.synth_frame(W, H, ps, t - 1, rects[t - 1])


def _check(cur, prev, W, H, T, r):
    want = S.mask(cur, prev, W, H, T, r)
    got = O.mask(cur, prev, W, H, T, r)
    assert np.array_equal(got, S.pack_bits(want)), (W, H, T, r)
    cg = O.cells(got, W, H)
    assert np.array_equal(cg, S.cells(want)), (W, H, T, r)
    assert O.extract_rois(cg, cap=65536) == S.rois(cg), (W, H, T, r)
    return cg


@pytest.mark.parametrize("r", [0, 1, 2, 5, 8])
def test_generator_frames_two_restatements_agree(r):
    cur, prev = _pair(1920, 1080, 1000 + r)
    cg = _check(cur, prev, 1920, 1080, 25, r)
    assert (cg != 0).any()


@pytest.mark.parametrize("W,H,T,r,density", [(640, 368, 25, 2, 0.002), (656, 200, 100, 3, 0.01),
                                             (1024, 75, 0, 1, 0.0005), (496, 300, 200, 0, 0.05)])
def test_random_frames_two_restatements_agree(W, H, T, r, density):
    """Sparse random foreground specks: many small components, blobs that
    touch diagonally, partial edge cells (H % 16 != 0), odd widths."""
    rng = np.random.default_rng(W * H + r)
    prev = rng.integers(0, 256, (H, 3 * W), dtype=np.uint8)
    cur = prev.copy()
    hit = rng.random((H, W)) < density
    ys, xs = np.nonzero(hit)
    for c in range(3):
        cur[ys, 3 * xs + c] = prev[ys, 3 * xs + c] ^ 0x80
    _check(cur, prev, W, H, T, r)


def test_4k_frame_two_restatements_agree():
    cur, prev = _pair(3840, 2160, 1234, roi_max_dim=480)
    _check(cur, prev, 3840, 2160, 25, 2)


def test_synth_rect_equals_frame_crops():
    W, H = 1280, 720
    cfg = O.gen_cfg(seed=5, n_frames=3, fps=30.0, frame_width=W, frame_height=H, roi_max_dim=300)
    _, rects = O.generate_trace(cfg)
    ps = O.derive_seed(5, "pixels")
    rng = np.random.default_rng(5)
    for t in (-1, 0, 1, 2):
        fr = O.synth_frame(W, H, ps, t, rects[t] if t >= 0 else [])
        for _ in range(20):
            w, h = int(rng.integers(1, 400)), int(rng.integers(1, 300))
            x, y = int(rng.integers(0, W - w + 1)), int(rng.integers(0, H - h + 1))
            got = O.synth_rect(W, H, ps, t, rects[t] if t >= 0 else [], (x, y, w, h))
            assert np.array_equal(got, fr[y:y + h, 3 * x:3 * (x + w)]), (t, x, y, w, h)
        canvas = np.zeros((200, 3 * 300), np.uint8)  # into a strided canvas view
        O.synth_rect(W, H, ps, t, rects[t] if t >= 0 else [], (100, 50, 120, 80),
                     out=canvas[10:90, 3 * 30:3 * 150])
        assert np.array_equal(canvas[10:90, 90:450], fr[50:130, 300:660])
        assert not canvas[:10].any() and not canvas[:, :90].any()
