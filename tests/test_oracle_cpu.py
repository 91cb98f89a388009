"""The oracle port (oracle/tangram_oracle.c) pinned against the reference.

* golden vectors produced by the reference itself (tests/golden/golden.json,
  made by tests/golden/make_golden.py from oracle/_ref) -- these run on any
  box;
* direct port-vs-reference comparisons when oracle/_ref/libtangram_ref.so is
  present (it is built wherever /root/reference exists and travels with the
  repo).
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O

need_ref = pytest.mark.skipif(not O.have_ref(), reason="reference build (oracle/_ref) absent")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tup(x):
    return [tuple(v) if isinstance(v, list) else v for v in x]


# ------------------------------------------------------------ rect level
def test_make_zones_golden(golden):
    z = golden["rect"]["zones"]
    assert O.make_zones(100, 100, 2, 2) == tup(z["100x100_2x2"])
    assert O.make_zones(101, 100, 2, 2) == tup(z["101x100_2x2"])
    assert O.make_zones(3840, 2160, 4, 4) == tup(z["3840x2160_4x4"])
    assert O.make_zones(1920, 1080, 6, 6) == tup(z["1920x1080_6x6"])


def test_partition_kats_golden(golden):
    for k in golden["rect"]["partition_kats"]:
        fid, w, h, gen, slo = k["frame"]
        got = O.partition(fid, w, h, gen, slo, *k["grid"], [tuple(r) for r in k["rois"]], k["bpp"],
                          k["first"])
        want = [dict(p, rect=tuple(p["rect"])) for p in k["patches"]]
        assert got == want


def test_partition_known_answers():
    # partition_test.cpp:79-99 and SPEC.md:125
    p = O.partition(7, 100, 100, 250000, 500000, 2, 2, [(30, 10, 30, 20), (5, 5, 10, 10)], 1.5, 40)
    assert len(p) == 1 and p[0]["rect"] == (5, 5, 55, 25) and p[0]["size_bytes"] == 2063
    assert p[0]["patch_id"] == 40 and p[0]["deadline_us"] == 750000


def test_partition_errors_golden(golden):
    errs = golden["rect"]["partition_errors"]
    with pytest.raises(O.OracleError) as e:
        O.partition(0, 100, 100, 0, 1, 2, 2, [(200, 200, 10, 10)], 1.5)
    assert str(e.value) == errs["outside"]
    with pytest.raises(O.OracleError) as e:
        O.partition(0, 3, 3, 0, 1, 4, 4, [], 1.5)
    assert str(e.value) == errs["finer"]


def test_stitch_kats_golden(golden):
    for k in golden["rect"]["stitch_kats"]:
        pl, nc, fr = O.stitch_all([tuple(q) for q in k["queue"]], *k["canvas"])
        assert pl == tup(k["placements"]) and nc == k["n_canvases"] and fr == tup(k["free"])
    with pytest.raises(O.OracleError) as e:
        O.stitch_all([(0, 101, 10)], 100, 100)
    assert str(e.value) == golden["rect"]["stitch_error"]


def test_stitch_c01_sets_golden(golden):
    for s in golden["rect"]["c01_sets"]:
        pl, nc, fr = O.stitch_all([tuple(q) for q in s["queue"]], 1024, 1024)
        assert pl == tup(s["placements"]) and nc == s["n_canvases"] and fr == tup(s["free"])


def test_generator_and_partition_golden(golden):
    for name, t in golden["rect"]["traces"].items():
        cfg = O.gen_cfg(**t["cfg"])
        t_us, frames = O.generate_trace(cfg)
        assert t_us == t["t_us"], name
        assert frames == [tup(f) for f in t["rois"]], name
        first = 0
        for i, rois in enumerate(frames):
            p = O.partition(i, cfg.frame_width, cfg.frame_height, t_us[i], 1_000_000, 4, 4, rois, 1.5,
                            first)
            first += len(p)
            assert [(q["patch_id"], *q["rect"], q["size_bytes"]) for q in p] == tup(t["patches"][i])


def test_generator_timestamps_and_bounds():
    # trace_test.cpp:160-205
    t_us, _ = O.generate_trace(O.gen_cfg(n_frames=5, fps=15.0))
    assert t_us[:4] == [0, 66667, 133333, 200000]
    _, frames = O.generate_trace(O.gen_cfg(n_frames=200, roi_count_min=5, roi_count_max=5,
                                           roi_max_dim=256, seed=4))
    for f in frames:
        assert len(f) == 5
        for (x, y, w, h) in f:
            assert 4 <= w <= 256 and 4 <= h <= 256 and x + w <= 1920 and y + h <= 1080


def test_rng_known_value():
    # std::mt19937_64 default-seed 10000th output is fixed by the C++ standard.
    r = O.Rng(5489)
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042


@need_ref
def test_port_equals_reference_random_stitch():
    rng = O.Rng(O.derive_seed(2026, "packing"))
    for _ in range(2000):
        n = rng.uniform_int(1, 40)
        q = [(i, rng.uniform_int(1, 200), rng.uniform_int(1, 200)) for i in range(n)]
        for cw, ch in ((256, 256), (300, 200)):
            assert O.stitch_all(q, cw, ch) == O.stitch_all(q, cw, ch, "ref")


@need_ref
def test_port_equals_reference_traces_and_partitions():
    for seed in range(1, 25):
        for kw in ({}, dict(frame_width=3840, frame_height=2160, n_frames=40, fps=30.0),
                   dict(roi_max_dim=1024, roi_proportion_mean=0.4, roi_count_max=30, n_frames=40)):
            cfg = O.gen_cfg(seed=seed, **kw)
            a, b = O.generate_trace(cfg), O.generate_trace(cfg, "ref")
            assert a == b
            for zx, zy in ((1, 1), (2, 2), (4, 4), (6, 6), (3, 5)):
                for i, rois in enumerate(a[1][:10]):
                    args = (i, cfg.frame_width, cfg.frame_height, a[0][i], 1000, zx, zy, rois, 1.5, 7)
                    assert O.partition(*args) == O.partition(*args, lib="ref")


@need_ref
def test_port_equals_reference_rng():
    import ctypes as C
    d = O.load("ref")
    n = 5000
    u = (C.c_uint64 * n)()
    dd = (C.c_double * n)()
    d.ref_rng_draws(17, 2, 3, 7, n, dd, u)
    r = O.Rng(17)
    assert all(r.uniform_int(3, 7) == u[i] for i in range(n))
    d.ref_rng_draws(13, 3, 100.0, 10.0, n, dd, u)
    r = O.Rng(13)
    assert all(r.normal(100.0, 10.0) == dd[i] for i in range(n))


# ------------------------------------------------------------ pixel level
def test_pixel_path_golden(golden):
    """Frozen pixel spec: the port reproduces its committed hashes (the rect
    stages inside were the reference's when the golden was made)."""
    for name, g in golden["pixel"].items():
        W, H, n, seed, radius = g["W"], g["H"], g["n"], g["seed"], g["radius"]
        cfg = O.gen_cfg(seed=seed, n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                        roi_max_dim=min(480, W, H))
        t_us, frames = O.generate_trace(cfg)
        ps = O.derive_seed(seed, "pixels")
        fr = [O.synth_frame(W, H, ps, -1, [])] + [O.synth_frame(W, H, ps, i, frames[i]) for i in range(n)]
        assert [sha(f) for f in fr] == g["frame_sha"], name
        params = dict(width=W, height=H, pitch=W * 3, threshold=25, radius=radius, zones_x=4,
                      zones_y=4, canvas_w=1024, canvas_h=1024, bytes_per_pixel=1.5,
                      slo_us=1_000_000, max_rois=1024, threads=2)
        res = O.process_frames(params, fr[1:], fr[:-1], list(range(n)), t_us, want_cells=True)
        assert [sha(O.mask(fr[i + 1], fr[i], W, H, 25, radius)) for i in range(n)] == g["mask_sha"]
        assert [sha(c) for c in res["cells"]] == g["cells_sha"], name
        assert [res["rois"][i, :res["n_rois"][i]].tolist() for i in range(n)] == g["rois"], name
        assert [[(q["patch_id"], *q["rect"], q["size_bytes"]) for q in p] for p in res["patch_list"]] \
            == [tup(p) for p in g["patches"]], name
        assert res["placement_list"] == [tup(p) for p in g["placements"]], name
        assert [sha(res["canvases"][k]) for k in range(res["total_canvases"])] == g["canvas_sha"], name


def test_raw_mask_is_union_of_consecutive_rects():
    """Synthetic-pixel design property: with r=0, fg = rects(t) ∪ rects(t-1)."""
    W, H = 640, 360
    cfg = O.gen_cfg(seed=3, n_frames=4, fps=30.0, frame_width=W, frame_height=H, roi_max_dim=200)
    _, frames = O.generate_trace(cfg)
    ps = O.derive_seed(3, "pixels")
    f = [O.synth_frame(W, H, ps, i, frames[i]) for i in range(4)]
    for t in range(1, 4):
        m = O.mask(f[t], f[t - 1], W, H, 25, 0)
        bits = np.unpackbits(m.view(np.uint8), bitorder="little").reshape(H, -1)[:, :W]
        exp = np.zeros((H, W), np.uint8)
        for (x, y, w, h) in frames[t] + frames[t - 1]:
            exp[y:y + h, x:x + w] = 1
        assert (bits == exp).all()


def test_round_trip_fixture_rois_equal_rects():
    """Cell-aligned, separated rects + static background + r=0: the
    extracted RoIs are exactly the rects (the end-to-end link between the
    pixel stages and the reference's rect-level inputs)."""
    W, H = 512, 256
    rects = [(16, 16, 64, 32), (128, 0, 48, 48), (256, 96, 160, 128), (32, 160, 16, 80)]
    ps = O.derive_seed(9, "pixels")
    bg = O.synth_frame(W, H, ps, -1, [])
    cur = O.synth_frame(W, H, ps, 0, rects)
    m = O.mask(cur, bg, W, H, 25, 0)
    rois = O.extract_rois(O.cells(m, W, H))
    assert sorted(rois) == sorted(rects)
