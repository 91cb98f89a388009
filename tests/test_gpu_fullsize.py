"""Parity at the BASELINE sizes the headline numbers are quoted on.

* config 2 -- one 4K camera, all 300 frames: every frame's cell grid, RoI
  list, patch list (every PatchMeta field), admission flags, placements and
  every canvas byte against the oracle pixel path run in 50-frame chunks
  (frames 100 and 200, where K1 restarts its frame chain, included);
* configs 3 (5 cameras x 300 4K frames) and 4 (64 cameras x 30 4K frames)
  through MultiCameraPath with the bench's batcher settings: every camera's
  RoIs against the oracle pixel path on oracle-synthesized frames, then the
  reference simulator tangram::run (sim.hpp:206-552, tangram policy, compiled
  as-is in oracle/_ref) on those RoIs: every invoke event, every arrival
  time, the whole scheduler event log byte for byte, and every canvas byte
  of every event against the reference's stitch_all of the event's patches
  filled with the oracle's pixels;
* config 5 at its densest point (rho = 0.59, roi_max_dim 1024): 8 cameras x
  60 frames through one per-frame pipeline run, every byte.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from paper_2404_09267_b200 import multicam as MC
from tests._helpers import GpuRun, oracle_params

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

W, H = 3840, 2160
THREADS = os.cpu_count() or 8
# bench.py's batcher setting: mu = 60 + 25k ms, 1e6 Mbps
# links, 80 GB GPU with a 4 GB model (76 canvases per batch)
SIM_PROFILE = [(k, 60.0 + 25.0 * k, 0.05 * (60.0 + 25.0 * k)) for k in (1, 2, 4, 8, 16, 32, 64)]
SIM = dict(bandwidth_mbps=1e6, gpu_memory_gb=80.0, model_size_gb=4.0)
TRIGGERS = {0: "deadline_timer", 1: "infeasible_arrival", 2: "memory_cap"}


def _patch_tuple(p):
    return (p.patch_id, p.source_frame_id, p.rect.x, p.rect.y, p.rect.w, p.rect.h,
            p.generation_time_us, p.slo_us, p.deadline_us, p.size_bytes)


def _opatch_tuple(p):
    return (p["patch_id"], p["source_frame_id"], *p["rect"], p["generation_time_us"], p["slo_us"],
            p["deadline_us"], p["size_bytes"])


def _compare_chunks(run, gpu, n, chunk=50):
    """Every frame of a GpuRun against the oracle pixel path, chunk by chunk
    (each chunk's first prev frame is the previous chunk's last frame)."""
    cells = run.pipe.cells(n)
    base = np.concatenate([[0], np.cumsum(gpu["n_canvases"])]).astype(np.int64)
    params = oracle_params(run.W, run.H, threads=THREADS, pitch=run.ring.pitch)
    first_id = 0
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        frames = [run.ring.download_frame(s) for s in range(a, b + 1)]
        ncv = int(base[b] - base[a])
        orc = O.process_frames(params, frames[1:], frames[:-1], list(range(a, b)), run.t_us[a:b],
                               first_id, want_cells=True, canvas_cap=max(1, ncv))
        assert orc["total_canvases"] == ncv, (a, b)
        for j, f in enumerate(range(a, b)):
            assert np.array_equal(cells[f], orc["cells"][j]), f
            assert gpu["n_rois"][f] == orc["n_rois"][j], f
            assert np.array_equal(gpu["rois"][f, :gpu["n_rois"][f]], orc["rois"][j, :orc["n_rois"][j]]), f
            assert [_patch_tuple(p) for p in gpu["patch_list"][f]] == \
                [_opatch_tuple(p) for p in orc["patch_list"][j]], f
            assert np.array_equal(gpu["admitted"][f, :gpu["n_patches"][f]],
                                  orc["admitted"][j, :orc["n_patches"][j]]), f
            assert gpu["placement_list"][f] == orc["placement_list"][j], f
            assert gpu["n_canvases"][f] == orc["n_canvases"][j], f
        first_id += int(sum(orc["n_patches"]))
        got = run.ctx.download(run.d_canvases + int(base[a]) * run.canvas_bytes,
                               (ncv, run.canvas[1], run.canvas[0] * 3), np.uint8)
        for c in range(ncv):
            assert np.array_equal(got[c], orc["canvases"][c]), (a, c)
        del frames, orc, got


def test_cfg2_all_300_frames_every_byte(ctx):
    run = GpuRun(ctx, W, H, 300, seed=1000, keep_mask=False,
                 trace_kw=dict(roi_proportion_mean=0.10, roi_max_dim=480))
    gpu = run.run()
    assert gpu["total_canvases"] > 600
    _compare_chunks(run, gpu, 300)
    run.close()


def test_cfg5_densest_point_every_byte(ctx):
    """rho = 0.59, roi_max_dim 1024, roi_count_max 24: 8 cameras x 60 frames
    as one camera-major per-frame run (K1 restarts its chain per camera)."""
    n, cams = 60, 8
    rings, cur, prev, gen, ts = [], [], [], [], []
    for c in range(cams):
        t_us, rects = A.generate_trace(n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                                       roi_proportion_mean=0.59, roi_max_dim=1024,
                                       roi_count_max=24, seed=1000 + c)
        ring = A.FrameRing(ctx, W, H, n)
        ring.synthesize(A.derive_seed(1000 + c, "pixels"), rects)
        rings.append(ring)
        cur += ring.slots[1:]
        prev += ring.slots[:-1]
        gen += list(t_us)
        ts.append(t_us)
    F = n * cams
    pipe = A.Pipeline(ctx, W, H, max_frames=F, max_canvases=F * 16)
    tabs = [ctx.malloc(8 * F) for _ in range(4)]
    for d, arr in zip(tabs, (np.array(cur, np.uint64), np.array(prev, np.uint64),
                             np.tile(np.arange(n, dtype=np.uint64), cams), np.array(gen, np.int64))):
        ctx.upload(d, arr)
    cb = pipe.canvas_bytes
    d_canv = ctx.malloc(cb * F * 16)
    pipe.run(F, *tabs, 0, d_canv)
    res = pipe.results(F)
    base = np.concatenate([[0], np.cumsum(res["n_canvases"])]).astype(np.int64)
    params = oracle_params(W, H, threads=THREADS)
    first_id = 0
    for c in range(cams):
        frames = [rings[c].download_frame(s) for s in range(n + 1)]
        a, b = c * n, (c + 1) * n
        ncv = int(base[b] - base[a])
        orc = O.process_frames(params, frames[1:], frames[:-1], list(range(n)), ts[c], first_id,
                               canvas_cap=max(1, ncv))
        assert orc["total_canvases"] == ncv
        for j in range(n):
            f = a + j
            assert np.array_equal(res["rois"][f, :res["n_rois"][f]], orc["rois"][j, :orc["n_rois"][j]])
            assert [_patch_tuple(p) for p in res["patch_list"][f]] == \
                [_opatch_tuple(p) for p in orc["patch_list"][j]]
            assert res["placement_list"][f] == orc["placement_list"][j]
        first_id += int(sum(orc["n_patches"]))
        got = ctx.download(d_canv + int(base[a]) * cb, (ncv, 1024, 3072), np.uint8)
        assert np.array_equal(got, orc["canvases"][:ncv]), c
    # the densest point rejects oversize patches (sim.hpp:262) and fills canvases
    assert int(res["admitted"].sum()) < int(res["n_patches"].sum())
    pipe.close()
    for r in rings:
        r.close()
    for p in tabs + [d_canv]:
        ctx.free(p)


def _oracle_camera(cam, n, trace_kw):
    """The oracle pixel path on oracle-synthesized frames of camera `cam`:
    (t_us, generator rects, extracted RoIs per frame)."""
    cfg = O.gen_cfg(seed=1000 + cam, n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                    **trace_kw)
    t_us, rects = O.generate_trace(cfg)
    frames = O.synth_frames(W, H, O.derive_seed(1000 + cam, "pixels"), rects, THREADS)
    orc = O.process_frames(oracle_params(W, H, threads=THREADS), frames[1:], frames[:-1],
                           list(range(n)), t_us, want_canvases=False)
    rois = [[tuple(r) for r in orc["rois"][f, :orc["n_rois"][f]].tolist()] for f in range(n)]
    return t_us, rects, rois


def _multicam_full(ctx, n_cams, n, trace_kw):
    path = MC.MultiCameraPath(ctx, list(range(n_cams)), W, H, n, SIM_PROFILE,
                              trace_kw=trace_kw, **SIM)
    path.sched.enable_log("tangram")
    _, n_events, n_canv = path.step()
    log = path.sched.take_log()
    ctx.stream_sync(path.stream)
    events = path.events()
    assert n_events == len(events) > 0 and n_canv == sum(e.batch_size for e in events)
    F = n_cams * n
    res = path.pipe.results(F, path.stream)
    # every camera's RoIs: GPU == oracle pixel path on oracle frames
    scenes, gen_rects = [], []
    for c in range(n_cams):
        t_us, rects, rois = _oracle_camera(c, n, trace_kw)
        assert t_us == path.t_us[c]
        for f in range(n):
            g = res["rois"][c * n + f, :res["n_rois"][c * n + f]].tolist()
            assert [tuple(r) for r in g] == rois[f], (c, f)
        scenes.append((t_us, rois))
        gen_rects.append(rects)
    # the reference simulator on those scenes
    ref = O.run_tangram(scenes, W, H, SIM_PROFILE, per_scene_link=True, **SIM)
    assert [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us, e.patch_ids)
            for e in events] == \
        [(e["fire_time_us"], TRIGGERS[e["trigger"]], e["batch_size"], e["estimated_slack_us"],
          e["patch_ids"]) for e in ref["events"]]
    adm = [i for i, a in enumerate(ref["admitted"]) if a]
    assert list(path.arrival) == [ref["arrival_us"][i] for i in adm]
    assert log == ref["log"]
    # patch table from the reference's own partition (global ids, sim.hpp:249-251)
    table, pid = {}, 0
    for c, (t_us, rois) in enumerate(scenes):
        for f in range(n):
            ps = O.partition(f, W, H, t_us[f], 1_000_000, 4, 4, rois[f], 1.5, pid, lib="ref")
            for p in ps:
                table[p["patch_id"]] = (c, f, p["rect"])
            pid += len(ps)
    # every event canvas: reference stitch_all of the event's patches, filled
    # with the oracle's pixels, against the bytes K5 wrote on the device
    seeds = [O.derive_seed(1000 + c, "pixels") for c in range(n_cams)]
    k = 0
    for e in events:
        q = [(i, table[i][2][2], table[i][2][3]) for i in e.patch_ids]
        pl, nc, _ = O.stitch_all(q, 1024, 1024, lib="ref")
        assert nc == e.batch_size
        want = np.zeros((nc, 1024, 3072), np.uint8)
        for (i, ci, x, y, w, h) in pl:
            c, f, r = table[i]
            O.synth_rect(W, H, seeds[c], f, gen_rects[c][f], (r[0], r[1], w, h),
                         out=want[ci, y:y + h, 3 * x:3 * (x + w)])
        got = ctx.download(path.d_canvases + k * path.canvas_bytes, (nc, 1024, 3072), np.uint8,
                           path.stream)
        assert np.array_equal(got, want), (e.fire_time_us, k)
        k += nc
    assert k == n_canv
    path.close()
    return len(events), n_canv


def test_cfg3_five_cameras_300_frames_vs_reference_run(ctx):
    n_ev, n_canv = _multicam_full(ctx, 5, 300, dict(roi_proportion_mean=0.10, roi_max_dim=480))
    assert n_ev > 5 and n_canv > 500


def test_cfg4_sixty_four_cameras_30_frames_vs_reference_run(ctx):
    n_ev, n_canv = _multicam_full(ctx, 64, 30, dict(roi_proportion_mean=0.10, roi_max_dim=480))
    assert n_ev > 50 and n_canv > 2000
