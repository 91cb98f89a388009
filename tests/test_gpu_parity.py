"""Parity of the B200 kernels with the oracle -- the gate for every claim.

Bit-exact everywhere (integer/byte work): masks, cell grids, RoI lists,
patch lists, admission, placements, free-rect lists (in the reference's list
order) and every canvas byte.  Rect-level outputs are additionally checked
against golden vectors produced by the reference itself.
"""
import hashlib
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from tests._helpers import GpuRun, oracle_patch_tuples, oracle_params, patch_tuples

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tup(x):
    return [tuple(v) if isinstance(v, list) else v for v in x]


# ============================================================ drop-in API
def test_partition_dropin_golden(ctx, golden):
    for k in golden["rect"]["partition_kats"]:
        fid, w, h, gen, slo = k["frame"]
        got = A.partition(A.FrameSpec(fid, w, h, gen, slo), A.PartitionConfig(*k["grid"]),
                          [tuple(r) for r in k["rois"]], k["bpp"], k["first"], ctx=ctx)
        want = [(p["patch_id"], p["source_frame_id"], *p["rect"], p["generation_time_us"],
                 p["slo_us"], p["deadline_us"], p["size_bytes"]) for p in k["patches"]]
        assert patch_tuples([got])[0] == want


def test_partition_dropin_errors(ctx, golden):
    errs = golden["rect"]["partition_errors"]
    with pytest.raises(A.InvalidArgument) as e:
        A.partition(A.FrameSpec(0, 100, 100, 0, 1), A.PartitionConfig(2, 2),
                    [(10, 10, 5, 5), (200, 200, 10, 10), (300, 300, 1, 1)], 1.5, ctx=ctx)
    assert str(e.value) == errs["outside"].replace("index 0", "index 1")
    with pytest.raises(A.InvalidArgument) as e:
        A.partition(A.FrameSpec(0, 3, 3, 0, 1), A.PartitionConfig(4, 4), [], 1.5, ctx=ctx)
    assert str(e.value) == errs["finer"]
    # the context is usable after an error
    assert len(A.partition(A.FrameSpec(0, 100, 100, 0, 1), A.PartitionConfig(2, 2),
                           [(1, 1, 3, 3)], 1.5, ctx=ctx)) == 1


def test_assign_rois_dropin(ctx):
    zones = A.make_zones(A.FrameSpec(0, 100, 100, 0, 1), A.PartitionConfig(2, 2))
    assert A.assign_rois([(30, 10, 30, 20)], zones, ctx=ctx)[0] == [0]
    assert A.assign_rois([(40, 10, 20, 10)], zones, ctx=ctx)[0] == [0]     # tie -> lowest zone
    assert A.assign_rois([(40, 40, 20, 20)], zones, ctx=ctx)[0] == [0]
    with pytest.raises(A.InvalidArgument, match=r"roi outside frame \(roi index 0\)"):
        A.assign_rois([(200, 200, 10, 10)], zones, ctx=ctx)


def test_partition_dropin_random_vs_reference_port(ctx):
    rng = O.Rng(O.derive_seed(5, "partition-gpu"))
    for it in range(300):
        W, H = rng.uniform_int(8, 4000), rng.uniform_int(8, 2200)
        zx, zy = rng.uniform_int(1, min(8, W)), rng.uniform_int(1, min(8, H))
        n = rng.uniform_int(0, 40)
        rois = []
        for _ in range(n):
            w, h = rng.uniform_int(1, W), rng.uniform_int(1, H)
            rois.append((rng.uniform_int(0, W - w), rng.uniform_int(0, H - h), w, h))
        bpp = [1.5, 1.0, 0.37, 3.0][it % 4]
        got = A.partition(A.FrameSpec(it, W, H, 1000 * it, 5000), A.PartitionConfig(zx, zy), rois,
                          bpp, 17 * it, ctx=ctx)
        want = O.partition(it, W, H, 1000 * it, 5000, zx, zy, rois, bpp, 17 * it)
        assert patch_tuples([got])[0] == oracle_patch_tuples([want])[0]


def test_partition_dropin_any_zone_grid(ctx):
    """The drop-in partition takes any zone grid, like the reference (the
    device accumulates zones 64 at a time): grids past 64 zones, against the
    port and the reference build."""
    rng = O.Rng(O.derive_seed(9, "partition-big-grids"))
    lib = "ref" if O.have_ref() else "port"
    for it, (zx, zy) in enumerate([(13, 5), (8, 9), (20, 20), (64, 2), (100, 30), (3, 200)]):
        W, H = max(zx, 1920), max(zy, 1080)
        n = rng.uniform_int(0, 120)
        rois = []
        for _ in range(n):
            w, h = rng.uniform_int(1, W // 3), rng.uniform_int(1, H // 3)
            rois.append((rng.uniform_int(0, W - w), rng.uniform_int(0, H - h), w, h))
        got = A.partition(A.FrameSpec(it, W, H, 1000 * it, 5000), A.PartitionConfig(zx, zy), rois,
                          1.5, 7 * it, ctx=ctx)
        want = O.partition(it, W, H, 1000 * it, 5000, zx, zy, rois, 1.5, 7 * it, lib=lib)
        assert len(got) > 0 or n == 0
        assert patch_tuples([got])[0] == oracle_patch_tuples([want])[0], (zx, zy)


def _stitch_tuples(res):
    pl = sorted([(p.patch_id, p.canvas_index, p.position.x, p.position.y, p.position.w,
                  p.position.h) for c in res.canvases for p in c.placements])
    fr = [(ci, r.x, r.y, r.w, r.h) for ci, c in enumerate(res.canvases) for r in c.free_rects]
    return pl, res.canvas_count(), fr


def test_stitch_dropin_golden(ctx, golden):
    for k in golden["rect"]["stitch_kats"] + [dict(s, canvas=(1024, 1024))
                                             for s in golden["rect"]["c01_sets"]]:
        q = [A.PatchMeta(pid, 0, A.Rect(0, 0, w, h)) for pid, w, h in k["queue"]]
        res = A.stitch_all(q, A.CanvasSpec(*k["canvas"]), ctx=ctx)
        pl, nc, fr = _stitch_tuples(res)
        assert pl == sorted(tup(k["placements"]))
        assert nc == k["n_canvases"]
        assert fr == tup(k["free"])  # reference list order, canvas by canvas
    with pytest.raises(A.InvalidArgument) as e:
        A.stitch_all([A.PatchMeta(0, 0, A.Rect(0, 0, 101, 10))], A.CanvasSpec(100, 100), ctx=ctx)
    assert str(e.value) == golden["rect"]["stitch_error"]
    assert A.stitch_all([], A.CanvasSpec(100, 100), ctx=ctx).empty()


def test_stitch_dropin_kat_values(ctx):
    # stitch_test.cpp:42-104
    q = [A.PatchMeta(i, 0, A.Rect(0, 0, w, h)) for i, (w, h) in enumerate([(60, 60), (40, 40)])]
    r = A.stitch_all(q, A.CanvasSpec(100, 100), ctx=ctx)
    assert r.canvas_count() == 1 and r.placement_index[1].position == A.Rect(60, 0, 40, 40)
    q = [A.PatchMeta(i, 0, A.Rect(0, 0, w, h)) for i, (w, h) in enumerate([(60, 60), (50, 50)])]
    r = A.stitch_all(q, A.CanvasSpec(100, 100), ctx=ctx)
    assert r.canvases[0].free_rects == [A.Rect(60, 0, 40, 100), A.Rect(0, 60, 60, 40)]
    assert A.canvas_efficiency(r) == [0.36, 0.25]


def wide_key_queue():
    """A queue whose best-fit winner sits on canvas 65540: canvas 0 offers a
    score-1 fit, canvases 1..65539 are full, canvas 65540 an exact (score 0)
    fit.  A (score, canvas, y, x) key with 16 canvas bits lets canvas 65540's
    high bit spill into the score and picks canvas 0 instead."""
    dims = [(60, 60)] + [(100, 100)] * 65539 + [(61, 61), (39, 39)]
    return [A.PatchMeta(i, 0, A.Rect(0, 0, w, h)) for i, (w, h) in enumerate(dims)]


def test_stitch_dropin_beyond_65535_canvases(ctx):
    q = wide_key_queue()
    r = A.stitch_all(q, A.CanvasSpec(100, 100), ctx=ctx)
    assert r.canvas_count() == 65541
    last = r.placement_index[len(q) - 1]
    assert (last.canvas_index, last.position) == (65540, A.Rect(61, 0, 39, 39))
    if O.have_ref():
        pl, nc, _ = O.stitch_all([(p.patch_id, p.rect.w, p.rect.h) for p in q[-3:]], 100, 100,
                                 lib="ref")
        assert nc == 2 and pl[-1][1:] == (1, 61, 0, 39, 39)  # same choice on a 2-canvas queue


def test_stitch_batch_c01_acceptance(ctx):
    """Acceptance C01 (acceptance_test.cpp:48-101): all 10,000 seeded sets,
    stitched in one batched launch (one warp per queue), every placement and
    free list equal to the oracle's."""
    from paper_2404_09267_b200 import _native as N
    rng = O.Rng(O.derive_seed(2026, "packing"))
    queues = []
    for _ in range(10_000):
        n = rng.uniform_int(1, 24)
        queues.append([(i, rng.uniform_int(16, 1024), rng.uniform_int(16, 1024)) for i in range(n)])
    offs = np.zeros(len(queues) + 1, np.int32)
    offs[1:] = np.cumsum([len(q) for q in queues])
    total = int(offs[-1])
    # tg_patch_meta as 8 int64 words: id, frame, (x|y<<32), (w|h<<32), gen, slo, ddl, bytes
    meta = np.zeros((total, 8), np.int64)
    k = 0
    for q in queues:
        for pid, w, h in q:
            meta[k, 0] = pid
            meta[k, 3] = h << 32 | w
            k += 1
    d_off, d_q = ctx.malloc(offs.nbytes), ctx.malloc(meta.nbytes)
    d_pl, d_nc = ctx.malloc(32 * total), ctx.malloc(4 * len(queues))
    d_fr, d_nf = ctx.malloc(24 * (2 * total + len(queues))), ctx.malloc(4 * len(queues))
    ctx.upload(d_off, offs)
    ctx.upload(d_q, meta)
    A.check(N.lib().tg_stitch_batch(ctx.handle, len(queues), total, d_off, d_q,
                                    N.tg_canvas_spec(1024, 1024, 1.0), d_pl, d_nc, d_fr, d_nf, None))
    ctx.stream_sync()
    pl = ctx.download(d_pl, (total, 8), np.int32)
    nc = ctx.download(d_nc, (len(queues),), np.int32)
    nf = ctx.download(d_nf, (len(queues),), np.int32)
    fr = ctx.download(d_fr, (2 * total + len(queues), 6), np.int32)
    for qi, q in enumerate(queues):
        want_pl, want_nc, want_fr = O.stitch_all(q, 1024, 1024)
        o = offs[qi]
        got_pl = [(int(pl[o + i, 0]), int(pl[o + i, 2]), int(pl[o + i, 3]), int(pl[o + i, 4]),
                   int(pl[o + i, 5]), int(pl[o + i, 6])) for i in range(len(q))]
        assert got_pl == want_pl, qi
        assert nc[qi] == want_nc
        base = 2 * o + qi
        f = fr[base:base + nf[qi]]
        got_fr = [(int(c), int(x), int(y), int(w), int(h))
                  for x, y, w, h, c, s in sorted(f.tolist(), key=lambda r: (r[4], r[5]))]
        assert got_fr == want_fr, qi
    for p in (d_off, d_q, d_pl, d_nc, d_fr, d_nf):
        ctx.free(p)


# ========================================================== pixel pipeline
def test_synth_matches_oracle(ctx):
    for (W, H, n, seed) in [(96, 64, 3, 5), (1920, 1080, 2, 1000), (208, 100, 2, 11)]:
        run = GpuRun(ctx, W, H, n, seed=seed, trace_kw=dict(roi_max_dim=min(480, W, H)))
        frames = run.host_frames()
        ps = O.derive_seed(seed, "pixels")
        assert sha(frames[0]) == sha(O.synth_frame(W, H, ps, -1, []))
        for i in range(n):
            rects = [(r.x, r.y, r.w, r.h) for r in run.rects[i]]
            assert sha(frames[i + 1]) == sha(O.synth_frame(W, H, ps, i, rects)), (W, H, i)
        run.close()


def _compare_full(run, gpu, orc, check_canvases=True):
    n = run.n
    # masks (when kept: the fused K1b then also writes the dilated mask) + cells
    if run.pipe.params.keep_mask:
        gm = run.pipe.mask(n)
        frames = run.host_frames()
        for i in range(n):
            om = O.mask(frames[i + 1], frames[i], run.W, run.H, run.threshold, run.radius)
            assert np.array_equal(gm[i], om), f"mask frame {i}"
    assert np.array_equal(run.pipe.cells(n), orc["cells"]), "cells"
    # RoIs in raster order of their first cell
    assert np.array_equal(gpu["n_rois"], orc["n_rois"])
    for i in range(n):
        assert np.array_equal(gpu["rois"][i, :gpu["n_rois"][i]], orc["rois"][i, :orc["n_rois"][i]]), i
    # patches, admission, placements
    assert patch_tuples(gpu["patch_list"]) == oracle_patch_tuples(orc["patch_list"])
    assert np.array_equal(gpu["admitted"][:, :], orc["admitted"])
    assert gpu["placement_list"] == orc["placement_list"]
    assert np.array_equal(gpu["n_canvases"], orc["n_canvases"])
    assert gpu["total_canvases"] == orc["total_canvases"]
    # free rects in reference list order
    zn = run.zones[0] * run.zones[1]
    for i in range(n):
        adm = [p for j, p in enumerate(orc["patch_list"][i]) if orc["admitted"][i, j]]
        if not adm:
            assert run.pipe.free_rects(i) == []
            continue
        _, _, want = O.stitch_all([(p["patch_id"], p["rect"][2], p["rect"][3]) for p in adm],
                                  *run.canvas)
        assert run.pipe.free_rects(i) == want, i
    assert zn > 0
    if check_canvases:
        got = run.canvases()
        want = orc["canvases"][:orc["total_canvases"]]
        assert got.shape == want.shape
        for k in range(got.shape[0]):
            assert np.array_equal(got[k], want[k]), f"canvas {k}"


@pytest.mark.parametrize("keep", [True, False])
def test_pipeline_cfg1_bit_exact(ctx, keep):
    """BASELINE config 1: one 1920x1080 camera, 30 frames, 4x4 grid, 1024^2
    canvases -- every intermediate and every canvas byte."""
    run = GpuRun(ctx, 1920, 1080, 30, seed=1000, keep_mask=keep)
    gpu = run.run()
    orc = run.oracle()
    _compare_full(run, gpu, orc)
    assert gpu["total_canvases"] > 0
    run.close()


def test_pipeline_cfg1_reference_rect_stages(ctx):
    """Same run, with the rect stages of the oracle path executed by the
    reference's own partition()/stitch_all() (oracle/_ref)."""
    if not O.have_ref():
        pytest.skip("oracle/_ref absent")
    run = GpuRun(ctx, 1920, 1080, 12, seed=1001)
    gpu = run.run()
    orc = run.oracle(lib="ref")
    assert patch_tuples(gpu["patch_list"]) == oracle_patch_tuples(orc["patch_list"])
    assert gpu["placement_list"] == orc["placement_list"]
    assert np.array_equal(run.canvases(), orc["canvases"][:orc["total_canvases"]])
    run.close()


@pytest.mark.parametrize("keep", [True, False])
def test_pipeline_cfg2_4k_bit_exact(ctx, keep):
    """BASELINE config 2 geometry (3840x2160, moderate density), first 20
    frames, every byte."""
    run = GpuRun(ctx, 3840, 2160, 20, seed=1000, keep_mask=keep)
    gpu = run.run()
    orc = run.oracle()
    _compare_full(run, gpu, orc)
    run.close()


@pytest.mark.slow
def test_pipeline_cfg2_full_300_frames(ctx):
    """All 300 frames of config 2: rect stages for every frame against the
    oracle's partition/stitch on the GPU's own RoIs, sampled frames fully
    against the oracle pixel path, and size-independent canvas properties
    for every canvas (exact tiling: placed bytes non-zero, free bytes zero)."""
    run = GpuRun(ctx, 3840, 2160, 300, seed=1000, keep_mask=False)
    gpu = run.run()
    first = 0
    for i in range(300):
        rois = [tuple(r) for r in gpu["rois"][i, :gpu["n_rois"][i]].tolist()]
        want = O.partition(i, 3840, 2160, run.t_us[i], 1_000_000, 4, 4, rois, 1.5, first)
        first += len(want)
        assert patch_tuples([gpu["patch_list"][i]])[0] == oracle_patch_tuples([want])[0]
        adm = [p for p in want if p["rect"][2] <= 1024 and p["rect"][3] <= 1024]
        if adm:
            pl, nc, _ = O.stitch_all([(p["patch_id"], p["rect"][2], p["rect"][3]) for p in adm],
                                     1024, 1024)
            assert gpu["placement_list"][i] == pl and gpu["n_canvases"][i] == nc
    # sampled frames through the whole oracle pixel path
    frames = {}
    idx = list(range(0, 300, 37))
    for i in idx:
        frames[i] = run.ring.download_frame(i)
        frames[i + 1] = run.ring.download_frame(i + 1)
    params = oracle_params(3840, 2160)
    orc = O.process_frames(params, [frames[i + 1] for i in idx], [frames[i] for i in idx], idx,
                           [run.t_us[i] for i in idx], 0, want_cells=True)
    cells = run.pipe.cells(300)
    base = np.concatenate([[0], np.cumsum(gpu["n_canvases"])])
    canv = run.canvases()
    ob = np.concatenate([[0], np.cumsum(orc["n_canvases"])])
    for j, i in enumerate(idx):
        assert np.array_equal(cells[i], orc["cells"][j])
        assert np.array_equal(gpu["rois"][i, :gpu["n_rois"][i]], orc["rois"][j, :orc["n_rois"][j]])
        for c in range(gpu["n_canvases"][i]):
            assert np.array_equal(canv[base[i] + c], orc["canvases"][ob[j] + c])
    # exact tiling on every canvas: synthetic pixels are never 0, so the
    # non-zero pattern must equal the union of placements.
    for i in range(300):
        for c in range(gpu["n_canvases"][i]):
            occ = np.zeros((1024, 1024), bool)
            for (_, ci, x, y, w, h) in gpu["placement_list"][i]:
                if ci == c:
                    assert not occ[y:y + h, x:x + w].any()
                    occ[y:y + h, x:x + w] = True
            nz = canv[base[i] + c].reshape(1024, 1024, 3).any(axis=2)
            assert np.array_equal(nz, occ), (i, c)
    run.close()


@pytest.mark.parametrize("density", [0.10, 0.40, 0.59])
def test_ccl_many_frames_vs_oracle_on_gpu_cells(ctx, density):
    """K2 over many dense 4K frames: the GPU's RoI boxes equal the oracle's
    components computed from the GPU's own cell grid (K1 is covered by the
    bit-exact tests; this isolates the concurrent union-find)."""
    run = GpuRun(ctx, 3840, 2160, 90, seed=2000, keep_mask=False,
                 trace_kw=dict(roi_proportion_mean=density, roi_max_dim=1024, roi_count_max=24))
    gpu = run.run()
    cells = run.pipe.cells(run.n)
    for i in range(run.n):
        want = O.extract_rois(cells[i])
        got = [tuple(r) for r in gpu["rois"][i, :gpu["n_rois"][i]].tolist()]
        assert got == want, i
    run.close()


def test_round_trip_fixture(ctx):
    """Cell-aligned separated rects, static background, r=0: the GPU RoIs
    equal the rects, so the patches equal the reference's partition() of
    those rects and the placements its stitch_all()."""
    rects = [[(16, 16, 64, 32), (128, 0, 48, 48), (256, 96, 160, 128), (32, 160, 16, 80),
              (480, 208, 32, 48)]]
    W, H = 512, 256
    run = GpuRun(ctx, W, H, 1, seed=9, radius=0, rects=rects)
    gpu = run.run()
    got = sorted(tuple(r) for r in gpu["rois"][0, :gpu["n_rois"][0]].tolist())
    assert got == sorted(rects[0])
    lib = "ref" if O.have_ref() else "port"
    want = O.partition(0, W, H, 0, 1_000_000, 4, 4, rects[0], 1.5, 0, lib=lib)
    assert patch_tuples(gpu["patch_list"])[0] == oracle_patch_tuples([want])[0]
    pl, nc, _ = O.stitch_all([(p["patch_id"], p["rect"][2], p["rect"][3]) for p in want], 1024, 1024,
                             lib=lib)
    assert gpu["placement_list"][0] == pl
    run.close()


@pytest.mark.parametrize("case", [
    dict(W=208, H=100, n=4, radius=2),                 # W % 32 == 16, H % 16 != 0
    dict(W=96, H=64, n=6, radius=3),
    dict(W=640, H=360, n=5, radius=0),
    dict(W=640, H=360, n=5, radius=8),
    dict(W=640, H=360, n=5, threshold=0),              # every noisy byte is foreground
    dict(W=640, H=360, n=5, threshold=200),            # the T >= 128 SWAR path
    dict(W=1280, H=720, n=4, zones=(1, 1)),
    dict(W=1280, H=720, n=4, zones=(8, 8)),
    dict(W=1280, H=720, n=4, zones=(10, 9)),            # past 64 zones: the 256-zone planner
    dict(W=1920, H=1088, n=3, zones=(16, 16), trace_kw=dict(roi_proportion_mean=0.3,
                                                            roi_count_max=40)),
    dict(W=1280, H=720, n=4, zones=(3, 5), canvas=(300, 200)),
    dict(W=640, H=352, n=3, pitch=640 * 3 + 64),       # padded rows
    dict(W=8192, H=48, n=3),                           # 4 K1 parts per row, 2 rows per item
    dict(W=2080, H=70, n=5),                           # 65 words: two uneven K1 parts
    dict(W=5008, H=40, n=3),                           # 5 K1 parts: 3 of 8 groups idle
    dict(W=16, H=8, n=4),                              # half a word, one partial cell row
    dict(W=32, H=3000, n=2),                           # tall: 750 row blocks, 47 K1b strips
    dict(W=1920, H=1080, n=6, trace_kw=dict(roi_proportion_mean=0.59, roi_max_dim=1080,
                                            roi_count_max=30)),  # dense, oversize patches
])
@pytest.mark.parametrize("keep", [True, False])
def test_pipeline_edge_cases(ctx, case, keep):
    case = dict(case)
    W, H, n = case.pop("W"), case.pop("H"), case.pop("n")
    tk = case.pop("trace_kw", dict(roi_max_dim=min(480, W, H)))
    run = GpuRun(ctx, W, H, n, seed=7, trace_kw=tk, keep_mask=keep, **case)
    gpu = run.run()
    orc = run.oracle()
    _compare_full(run, gpu, orc)
    run.close()


def test_pipeline_broken_frame_chains(ctx):
    """prev[i] need not be cur[i-1]: K1 restarts its frame chain wherever the
    pointer tables break it (a prev that is some other frame, the frame itself,
    the background slot)."""
    W, H, n = 1280, 720, 7
    run = GpuRun(ctx, W, H, n, seed=11, trace_kw=dict(roi_max_dim=400))
    slots = run.ring.slots
    cur_slot = [i + 1 for i in range(n)]
    prev_slot = [0, 1, 0, 3, 5, 5, 2]  # chain, chain, break, chain, self, chain, break
    d_cur, d_prev = ctx.malloc(8 * n), ctx.malloc(8 * n)
    ctx.upload(d_cur, np.array([slots[s] for s in cur_slot], np.uint64))
    ctx.upload(d_prev, np.array([slots[s] for s in prev_slot], np.uint64))
    run.pipe.run(n, d_cur, d_prev, run.d_ids, run.d_gen, 0, run.d_canvases)
    gpu = run.pipe.results(n)
    frames = run.host_frames()
    gm = run.pipe.mask(n)
    for i in range(n):
        om = O.mask(frames[cur_slot[i]], frames[prev_slot[i]], W, H, run.threshold, run.radius)
        assert np.array_equal(gm[i], om), f"mask frame {i}"
    params = oracle_params(W, H, run.radius, run.threshold, run.zones, run.canvas, run.max_rois,
                           pitch=run.ring.pitch)
    orc = O.process_frames(params, [frames[s] for s in cur_slot], [frames[s] for s in prev_slot],
                           list(range(n)), run.t_us, 0, want_canvases=True, want_cells=True)
    assert np.array_equal(run.pipe.cells(n), orc["cells"])
    assert patch_tuples(gpu["patch_list"]) == oracle_patch_tuples(orc["patch_list"])
    assert gpu["placement_list"] == orc["placement_list"]
    assert gpu["total_canvases"] == orc["total_canvases"]
    got = ctx.download(run.d_canvases, (gpu["total_canvases"], 1024, 3072), np.uint8)
    assert np.array_equal(got, orc["canvases"][:orc["total_canvases"]])
    for d in (d_cur, d_prev):
        ctx.free(d)
    run.close()


def test_pipeline_empty_and_full_motion(ctx):
    # no RoIs at all: no patches, no canvases
    run = GpuRun(ctx, 640, 480, 3, rects=[[], [], []])
    gpu = run.run()
    # frame 0 differs from the background only by noise -> nothing
    assert gpu["n_rois"].tolist() == [0, 0, 0] and gpu["total_canvases"] == 0
    run.close()
    # the whole frame moves: one giant RoI, a patch larger than the canvas
    # is rejected (sim.hpp:262) and never stitched.
    run = GpuRun(ctx, 1280, 1280, 2, rects=[[(0, 0, 1280, 1280)], [(0, 0, 1280, 1280)]])
    gpu = run.run()
    assert gpu["n_rois"].tolist() == [1, 1]
    assert gpu["admitted"][:, 0].tolist() == [0, 0] and gpu["total_canvases"] == 0
    _compare_full(run, gpu, run.oracle())
    run.close()


def test_pipeline_capacity_errors(ctx):
    run = GpuRun(ctx, 640, 480, 4, max_rois=2, trace_kw=dict(roi_count_min=8, roi_count_max=12,
                                                            roi_max_dim=60))
    with pytest.raises(A.CapacityError, match="roi capacity"):
        run.run()
    run.close()
    run = GpuRun(ctx, 1920, 1080, 8, max_canvases=1)
    with pytest.raises(A.CapacityError, match="canvas capacity"):
        run.run()
    run.close()


def test_pipeline_argument_validation(ctx):
    """tg_pipeline_create and the stages reject bad geometry / capacities
    with tg_last_error messages (no device work is launched), and the
    context stays usable."""
    from paper_2404_09267_b200 import _native as N
    bad = [
        (dict(W=100, H=64), "multiple of 16"),
        (dict(W=8208, H=64), "multiple of 16"),
        (dict(W=640, H=0), "multiple of 16"),
        (dict(W=640, H=70000), "height must be <= 65535"),
        (dict(W=640, H=64, pitch=640 * 3 - 16), "pitch"),
        (dict(W=640, H=64, pitch=640 * 3 + 8), "pitch"),
        (dict(W=640, H=64, threshold=256), "threshold"),
        (dict(W=640, H=64, dilate_radius=9), "dilate radius"),
        (dict(W=640, H=32, zones=(1, 40)), "zone grid finer than frame"),
        (dict(W=640, H=64, zones=(20, 13)), "pipeline limit"),
        (dict(W=640, H=64, canvas=(0, 1024)), "canvas dimensions"),
        (dict(W=640, H=64, max_frames=0), "capacities"),
        (dict(W=8192, H=2064), "more than 65535"),
        (dict(W=640, H=64, max_rois_per_frame=100000), "max_rois_per_frame too large"),
        (dict(W=640, H=64, max_frames=600000), "below 2\\^23"),
    ]
    for kw, msg in bad:
        kw = dict(kw)
        W, H = kw.pop("W"), kw.pop("H")
        kw.setdefault("max_frames", 2)
        with pytest.raises(A.InvalidArgument, match=msg):
            A.Pipeline(ctx, W, H, **kw)
    run = GpuRun(ctx, 640, 64, 2, seed=5, trace_kw=dict(roi_max_dim=60))
    lib = N.lib()
    with pytest.raises(A.InvalidArgument, match="n_frames must be in"):
        A.check(lib.tg_pipeline_stage_mask(run.pipe.handle, 3, run.d_cur, run.d_prev, None))
    with pytest.raises(A.InvalidArgument, match="null frame pointer table"):
        A.check(lib.tg_pipeline_stage_mask(run.pipe.handle, 2, None, None, None))
    gpu = run.run()  # still fine afterwards
    _compare_full(run, gpu, run.oracle())
    run.close()


def test_pipeline_graph_replay_and_patch_id_base(ctx):
    run = GpuRun(ctx, 1920, 1080, 8, seed=3, first_patch_id=1000)
    gpu = run.run()
    first = run.canvases()
    run.ctx.memset(run.d_canvases, 0, run.canvas_bytes * run.max_canvases)
    g = run.pipe.graph(run.n, run.d_cur, run.d_prev, run.d_ids, run.d_gen, 1000, run.d_canvases)
    g.launch()
    g.launch()
    again = run.pipe.results(run.n)
    assert again["placement_list"] == gpu["placement_list"]
    assert np.array_equal(run.canvases(), first)
    assert gpu["patch_list"][0][0].patch_id == 1000
    g.close()
    run.close()


def test_cpp_dropin_binary():
    """The C++ drop-in headers (include/tangram/*.hpp) compile against the
    reference's own test expectations and run on the GPU."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "dropin_test"])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout


def test_cpp_pipeline_binary():
    """The whole path from C++ through the C ABI alone (tests/cpp/
    pipeline_test.cpp): device frames -> tg_pipeline_run -> descriptors ->
    tg_batcher_schedule -> event canvases, against the C oracle."""
    exe = os.path.join(ROOT, "tests", "cpp", "pipeline_test")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "pipeline_test"])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout


def test_gather_repeats_and_rewrites_every_byte(ctx):
    """K5 claims units from a device counter that its last CTA resets: a
    second gather after one plan (no scan in between) must rewrite every
    canvas byte identically, including over garbage."""
    from paper_2404_09267_b200 import _native as N
    run = GpuRun(ctx, 1920, 1080, 12, seed=1004, trace_kw=dict(roi_proportion_mean=0.2))
    run.run()
    first = run.canvases()
    total = run.res["total_canvases"]
    assert total > 0
    for _ in range(3):
        run.ctx.memset(run.d_canvases, 0x5A, run.canvas_bytes * total)
        A.check(N.lib().tg_pipeline_stage_gather(run.pipe.handle, run.n, run.d_cur,
                                                 run.d_canvases, None))
        run.ctx.stream_sync()
        assert np.array_equal(run.canvases(), first)
    orc = run.oracle()
    assert np.array_equal(first, orc["canvases"][:total])
    run.close()


@pytest.mark.parametrize("keep", [True, False])
def test_two_launch_mask_path_stage_by_stage(ctx, keep):
    """The mask stage as two launches (K1 tg_pipeline_stage_mask_fg, then
    K1b tg_pipeline_stage_mask_cells: the fallback tg_pipeline_stage_mask
    takes when the cooperative launch cannot be co-scheduled), followed by
    the plan and gather stages called one by one: bit-exact like the fused
    tg_pipeline_run."""
    from paper_2404_09267_b200 import _native as N
    lib = N.lib()
    run = GpuRun(ctx, 1920, 1080, 9, seed=1006, keep_mask=keep,
                 trace_kw=dict(roi_proportion_mean=0.2))
    ctx.memset(run.d_canvases, 0x5A, run.canvas_bytes * run.max_canvases)
    A.check(lib.tg_pipeline_stage_mask_fg(run.pipe.handle, run.n, run.d_cur, run.d_prev, None))
    A.check(lib.tg_pipeline_stage_mask_cells(run.pipe.handle, run.n, None))
    A.check(lib.tg_pipeline_stage_plan(run.pipe.handle, run.n, run.d_ids, run.d_gen,
                                       run.first_patch_id, None))
    A.check(lib.tg_pipeline_stage_gather(run.pipe.handle, run.n, run.d_cur, run.d_canvases, None))
    run.ctx.stream_sync()
    run.res = run.pipe.results(run.n)
    _compare_full(run, run.res, run.oracle())
    run.close()


@pytest.mark.parametrize("case", [
    dict(W=208, H=100, n=4, radius=2),                 # W % 32 == 16, H % 16 != 0
    dict(W=96, H=64, n=6, radius=3),
    dict(W=640, H=360, n=5, radius=0),
    dict(W=640, H=360, n=5, radius=8),
    dict(W=640, H=360, n=5, threshold=0),              # every noisy byte is foreground
    dict(W=992, H=77, n=4),                            # 31 words: one 32-word part
    dict(W=8192, H=48, n=3),                           # 4 K1 parts per row
    dict(W=2080, H=70, n=5),                           # 65 words: parts of 64 + 1 (sparse)
    dict(W=5008, H=40, n=3),
    dict(W=16, H=8, n=4),                              # half a word
    dict(W=32, H=3000, n=2),                           # tall
    dict(W=3840, H=2160, n=3),                         # 4K: parts of 64 + 56 words (sparse)
])
@pytest.mark.parametrize("keep", [True, False])
def test_two_launch_mask_path_over_stale_bitmap(ctx, case, keep):
    """The split K1 / K1b launches (configs 3/4 run them; with TG_K1_SPARSE
    K1 stores only the raw sectors holding foreground plus per-row word
    flags) at edge geometries, over a raw bitmap a first pass on other,
    dense frames left full of stale bits: bit-exact vs the oracle."""
    from paper_2404_09267_b200 import _native as N
    lib = N.lib()
    case = dict(case)
    W, H, n = case.pop("W"), case.pop("H"), case.pop("n")
    run = GpuRun(ctx, W, H, n, seed=7, trace_kw=dict(roi_max_dim=min(480, W, H)),
                 keep_mask=keep, **case)
    junk = GpuRun(ctx, W, H, n, seed=99, pitch=run.ring.pitch,
                  trace_kw=dict(roi_proportion_mean=0.59, roi_max_dim=min(W, H), roi_count_max=30))
    h = run.pipe.handle
    A.check(lib.tg_pipeline_stage_mask_fg(h, n, junk.d_cur, junk.d_prev, None))
    A.check(lib.tg_pipeline_stage_mask_cells(h, n, None))
    A.check(lib.tg_pipeline_stage_mask_fg(h, n, run.d_cur, run.d_prev, None))
    A.check(lib.tg_pipeline_stage_mask_cells(h, n, None))
    A.check(lib.tg_pipeline_stage_plan(h, n, run.d_ids, run.d_gen, run.first_patch_id, None))
    A.check(lib.tg_pipeline_stage_gather(h, n, run.d_cur, run.d_canvases, None))
    run.ctx.stream_sync()
    run.res = run.pipe.results(n)
    _compare_full(run, run.res, run.oracle())
    junk.close()
    run.close()


@pytest.mark.parametrize("M,band", [(300, 0), (320, 0), (320, 1), (320, 8), (320, 512)])
def test_stitch_gather_explicit_plan(ctx, M, band):
    """tg_stitch_gather (A13 on a caller-built plan): the oracle's stitch of
    patches cut from several frames -> placement jobs + zero jobs for the
    final free rects; every canvas byte equals the SURVEY A13 fill
    canvas[py+v][(px+u)*3+c] = frame[ry+v][(rx+u)*3+c], uncovered = 0,
    over canvases pre-filled with garbage.  Malformed plans fail loudly.
    M = 300 takes K5's rect-by-rect path (rows not 16-byte multiples), 320
    its TMA pipeline; band = TG_OPT_GATHER_BAND (0 = automatic, 512 = one
    unit per canvas)."""
    import ctypes as C

    from paper_2404_09267_b200 import _native as N
    W, H, n, Nh = 640, 360, 4, 200
    with pytest.raises(A.InvalidArgument, match="gather band out of range"):
        A.check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_BAND, -1))
    A.check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_BAND, band))
    run = GpuRun(ctx, W, H, n, seed=1007, trace_kw=dict(roi_max_dim=200))
    frames = run.host_frames()
    rng = O.Rng(O.derive_seed(1007, "stitch-gather"))
    src = {}
    queue = []
    for pid in range(40):
        w, h = rng.uniform_int(1, M), rng.uniform_int(1, Nh)
        f = rng.uniform_int(0, n - 1)
        src[pid] = (f, rng.uniform_int(0, W - w), rng.uniform_int(0, H - h))
        queue.append((pid, w, h))
    pl, nc, free = O.stitch_all(queue, M, Nh)
    jobs, offs = [], [0]
    for c in range(nc):
        for pid, ci, x, y, w, h in pl:
            if ci == c:
                f, rx, ry = src[pid]
                jobs.append(N.tg_gather_job(N.tg_rect(x, y, w, h), f, rx, ry))
        for ci, x, y, w, h in free:
            if ci == c:
                jobs.append(N.tg_gather_job(N.tg_rect(x, y, w, h), -1, 0, 0))
        offs.append(len(jobs))
    want = np.zeros((nc, Nh, M * 3), np.uint8)
    for pid, ci, x, y, w, h in pl:
        f, rx, ry = src[pid]
        want[ci, y:y + h, 3 * x:3 * (x + w)] = frames[f + 1][ry:ry + h, 3 * rx:3 * (rx + w)]
    cbytes = M * Nh * 3
    d_canv = ctx.malloc(cbytes * nc)
    ctx.memset(d_canv, 0xC3, cbytes * nc)
    c_jobs = (N.tg_gather_job * len(jobs))(*jobs)
    c_offs = (C.c_int32 * len(offs))(*offs)
    spec = N.tg_canvas_spec(M, Nh, 1.0)
    A.check(N.lib().tg_stitch_gather(ctx.handle, c_jobs, len(jobs), c_offs, nc, spec, run.d_cur,
                                     run.ring.pitch, d_canv, None))
    ctx.stream_sync()
    got = ctx.download(d_canv, (nc, Nh, M * 3), np.uint8)
    assert nc >= 2
    for k in range(nc):
        assert np.array_equal(got[k], want[k]), f"canvas {k}"
    bad = (C.c_int32 * 2)(0, len(jobs) + 1)
    with pytest.raises(A.InvalidArgument, match="bad job offsets"):
        A.check(N.lib().tg_stitch_gather(ctx.handle, c_jobs, len(jobs), bad, 1, spec, run.d_cur,
                                         run.ring.pitch, d_canv, None))
    with pytest.raises(A.InvalidArgument, match="pitch must be a multiple of 16"):
        A.check(N.lib().tg_stitch_gather(ctx.handle, c_jobs, len(jobs), c_offs, nc, spec, run.d_cur,
                                         run.ring.pitch + 8, d_canv, None))
    ctx.free(d_canv)
    A.check(N.lib().tg_ctx_set_option(ctx.handle, N.TG_OPT_GATHER_BAND, 0))
    run.close()


def test_c07_granularity_on_device_partition(ctx):
    """acceptance_test.cpp:310-347 with the device partition (drop-in
    tg_partition): finer zone grids transmit no more bytes; and every frame's
    patches equal the reference port's."""
    from tests.test_geometry_cpu import c07_means, check_c07

    def pb(i, W, H, t, z, rois):
        got = A.partition(A.FrameSpec(i, W, H, t, 1_000_000), A.PartitionConfig(z, z),
                          [A.Rect(*r) for r in rois], 1.5, 0, ctx=ctx)
        if i % 17 == 0:  # sampled frames: field-for-field against the port
            want = O.partition(i, W, H, t, 1_000_000, z, z, rois, 1.5, 0)
            assert patch_tuples([got]) == oracle_patch_tuples([want])
        return float(sum(p.size_bytes for p in got))

    check_c07(*c07_means(pb))


def test_chunked_runs_continue_patch_ids_on_device(ctx):
    """The e2e path's chunked streaming: runs over consecutive chunks with
    first_patch_id = TG_CONTINUE_PATCH_IDS number patches exactly as one run
    over all frames (sim.hpp:249-251), with no host round trip, and every
    chunk's canvases equal the single run's."""
    n, chunk = 20, 7
    run = GpuRun(ctx, 1280, 720, n, seed=1010, trace_kw=dict(roi_proportion_mean=0.2),
                 keep_mask=False)
    whole = run.run()
    want_canv = run.canvases()
    got_patches, got_pl, got_canv = [], [], []
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        first = 0 if c0 == 0 else 0xFFFFFFFFFFFFFFFF  # TG_CONTINUE_PATCH_IDS
        run.pipe.run(m, run.d_cur + 8 * c0, run.d_prev + 8 * c0, run.d_ids + 8 * c0,
                     run.d_gen + 8 * c0, first, run.d_canvases)
        res = run.pipe.results(m)
        got_patches += patch_tuples(res["patch_list"])
        got_pl += res["placement_list"]
        got_canv.append(run.ctx.download(run.d_canvases, (res["total_canvases"], 1024, 1024 * 3),
                                         np.uint8))
    assert got_patches == patch_tuples(whole["patch_list"])
    # placements: same patch ids and positions; canvas indices are per frame
    assert got_pl == whole["placement_list"]
    assert np.array_equal(np.concatenate(got_canv), want_canv)
    run.close()


def test_plan_look_back_survives_epoch_wrap(ctx):
    """Look-back words carry a 16-bit launch epoch and are zeroed every 32768
    launches: after more than 65536 plan launches on one pipeline, patch ids
    and canvas numbering are still exact (a stale word from 65536 launches
    ago must never pass for a fresh one)."""
    from paper_2404_09267_b200 import _native as N
    run = GpuRun(ctx, 640, 368, 12, seed=77, keep_mask=False, trace_kw=dict(roi_max_dim=200))
    want = run.run()
    lib = N.lib()
    for _ in range(65536 + 7):  # plan stage alone, one frame: every launch moves the epoch
        A.check(lib.tg_pipeline_stage_plan(run.pipe.handle, 1, run.d_ids, run.d_gen, 0, None))
    got = run.run()
    assert got["patch_list"] == want["patch_list"]
    assert got["placement_list"] == want["placement_list"]
    assert got["total_canvases"] == want["total_canvases"]
    run.close()


def test_cpp_dropin_per_frame_loop_matches_reference_build():
    """A reference caller's per-frame loop (partition + stitch_all through
    include/tangram, tests/cpp/dropin_bench.cpp) gives the same placements
    as the same source built against the reference headers."""
    cpp = os.path.join(ROOT, "tests", "cpp")
    subprocess.check_call(["make", "-s", "-C", cpp, "dropin_bench"])
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", cpp, "dropin_bench_ref"])

    def run(exe):
        out = subprocess.run([os.path.join(cpp, exe), "120"], capture_output=True, text=True,
                             timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr
        return out.stdout.splitlines()[0]
    ours = run("dropin_bench")
    assert ours.startswith("checksum ")
    if os.path.exists(os.path.join(cpp, "dropin_bench_ref")):
        assert ours == run("dropin_bench_ref")


@pytest.mark.parametrize("radius", [0, 2])
def test_mask_threshold_boundaries_random_bytes(ctx, radius):
    """The per-pixel foreground test (max over channels of |cur - prev| > T,
    K1's VIMNMX3 form and both SWAR threshold paths) against the oracle on
    frames whose byte differences sit on and around every tested threshold
    and the 7-bit boundary, for T across [0, 255]."""
    from paper_2404_09267_b200 import _native as N
    W, H, n = 640, 48, 3
    rng = np.random.default_rng(7 + radius)
    for T in (0, 1, 24, 25, 26, 126, 127, 128, 129, 200, 254, 255):
        ring = A.FrameRing(ctx, W, H, n)
        pitch = ring.pitch
        base = rng.integers(0, 256, size=(H, pitch), dtype=np.int32)
        frames = [base]
        for _ in range(n):
            d = rng.choice(np.array([0, 1, T - 1, T, T + 1, 127, 128, 255]), size=(H, pitch))
            sign = rng.choice(np.array([-1, 1]), size=(H, pitch))
            nxt = np.clip(frames[-1] + sign * d, 0, 255)
            sparse = rng.random((H, pitch)) < 0.5  # half the bytes unchanged
            frames.append(np.where(sparse, frames[-1], nxt))
        frames = [f.astype(np.uint8) for f in frames]
        for i, f in enumerate(frames):
            ctx.upload(ring.slots[i], np.ascontiguousarray(f))
        pipe = A.Pipeline(ctx, W, H, dilate_radius=radius, threshold=T, max_frames=n,
                          keep_mask=1, max_canvases=64, pitch=pitch)
        d_cur, d_prev = ring.tables()
        A.check(N.lib().tg_pipeline_stage_mask(pipe.handle, n, d_cur, d_prev, None))
        ctx.synchronize()
        gm = pipe.mask(n)
        cells = pipe.cells(n)
        for i in range(n):
            om = O.mask(frames[i + 1], frames[i], W, H, T, radius)
            assert np.array_equal(gm[i], om), (T, radius, i)
            assert np.array_equal(cells[i], O.cells(om, W, H)), (T, radius, i)
        pipe.close()
        ring.close()
