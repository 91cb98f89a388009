"""Configs 3/4 on the device: cameras -> K1-K4 -> descriptors -> SLO batcher
-> event canvases, against the reference's own simulator.

The RoIs the GPU extracts from pixels are fed, as trace rects, to the
reference's tangram::run(): it partitions them itself, models the uplinks
and drives its SloScheduler.  Every invoke it logs must equal ours, and every
canvas byte we write must equal a host fill of that event's placements from
the same frames.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from paper_2404_09267_b200 import multicam as MC

pytestmark = pytest.mark.gpu

PROFILE = [(1, 60.0, 3.0), (2, 85.0, 4.0), (4, 135.0, 6.0), (8, 235.0, 10.0)]


@pytest.mark.parametrize("cams,W,H,n,bw,link", [
    ([0, 1, 2], 1920, 1080, 12, 80.0, True),
    ([3, 4, 5, 6, 7], 3840, 2160, 6, 20.0, True),
    ([0, 1], 1920, 1080, 10, 40.0, False),
])
def test_multicam_events_and_canvases_match_reference(ctx, cams, W, H, n, bw, link):
    path = MC.MultiCameraPath(ctx, cams, W, H, n, PROFILE, bandwidth_mbps=bw, per_camera_link=link,
                              trace_kw=dict(roi_proportion_mean=0.15))
    path.sched.enable_log("tangram")
    desc, n_events, n_canvases = path.step()
    log = path.sched.take_log()
    ctx.stream_sync(path.stream)
    assert n_events > 0 and n_canvases > 0
    events = path.events()
    # the GPU's RoIs, as the reference simulator's input scenes
    scenes, frames = [], []
    for k, c in enumerate(cams):
        res = path.camera_results(k)
        rois = [[tuple(r) for r in res["rois"][f, :res["n_rois"][f]].tolist()] for f in range(n)]
        scenes.append((path.t_us[k], rois))
        frames.append([path.rings[k].download_frame(s) for s in range(n + 1)])
    if O.have_ref():
        ref = O.run_tangram(scenes, W, H, PROFILE, bandwidth_mbps=bw, per_scene_link=link)
        names = {0: "deadline_timer", 1: "infeasible_arrival", 2: "memory_cap"}
        assert [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us, e.patch_ids)
                for e in events] == \
            [(e["fire_time_us"], names[e["trigger"]], e["batch_size"], e["estimated_slack_us"],
              e["patch_ids"]) for e in ref["events"]]
        adm_ids = [i for i, a in enumerate(ref["admitted"]) if a]
        assert list(path.arrival) == [ref["arrival_us"][i] for i in adm_ids]
        assert log == ref["log"]  # the whole scheduler event log, byte for byte
    # canvas bytes: host fill of every event canvas from the same frames
    plan = path._last
    by_id = {int(p["patch_id"]): (int(s), p) for p, s in zip(plan["patches"], plan["src"])}
    got = path.canvases(n_canvases)
    k = 0
    for e in events:
        for cv in e.stitch.canvases:
            want = np.zeros((1024, 1024 * 3), np.uint8)
            for pl in cv.placements:
                src, p = by_id[pl.patch_id]
                cam_slot, slot = divmod(src, n + 1)
                fr = frames[cam_slot][slot]
                x, y, w, h = pl.position.x, pl.position.y, pl.position.w, pl.position.h
                want[y:y + h, 3 * x:3 * (x + w)] = fr[p["y"]:p["y"] + h, 3 * p["x"]:3 * (p["x"] + w)]
            assert np.array_equal(got[k], want), (k, e.fire_time_us)
            k += 1
    assert k == n_canvases
    path.close()


def test_pipelined_passes_match_a_single_step(ctx):
    """run_pipelined (host batcher of pass i beside the planes of pass i+1,
    K5 on its own stream) leaves the same events and canvases as step()."""
    cams = [0, 1, 2, 3]
    path = MC.MultiCameraPath(ctx, cams, 1920, 1080, 8, PROFILE, bandwidth_mbps=40.0,
                              trace_kw=dict(roi_proportion_mean=0.15))
    _, n_events, n_canv = path.step()
    ctx.stream_sync(path.stream)
    want_ev = [(e.fire_time_us, e.trigger, e.batch_size, e.patch_ids) for e in path.events()]
    want = path.canvases(n_canv)
    got_n = path.run_pipelined(3)
    ctx.stream_sync(path.stream)
    assert got_n == n_canv
    assert [(e.fire_time_us, e.trigger, e.batch_size, e.patch_ids) for e in path.events()] == want_ev
    assert np.array_equal(path.canvases(n_canv), want)
    path.close()


def test_event_subsets_partition_the_canvases(ctx):
    """tg_batcher_gather_events(first, stride) writes exactly the canvases of
    events first, first+stride, ... in event order."""
    import ctypes as C

    from paper_2404_09267_b200 import _native as N
    path = MC.MultiCameraPath(ctx, [0, 1, 2], 1920, 1080, 10, PROFILE, bandwidth_mbps=40.0,
                              trace_kw=dict(roi_proportion_mean=0.2))
    _, n_events, n_canv = path.step()
    ctx.stream_sync(path.stream)
    every = path.canvases(n_canv)
    sizes = [e.batch_size for e in path.events()]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for stride in (2, 3):
        for first in range(stride):
            n = C.c_int64()
            A.check(N.lib().tg_batcher_gather_events(ctx.handle, path.sched.handle, first, stride,
                                                     path.d_frames, 3 * path.W, path.d_canvases,
                                                     path.canvas_cap, C.byref(n), path.stream))
            ctx.stream_sync(path.stream)
            want = [every[offs[e]:offs[e + 1]] for e in range(first, len(sizes), stride)]
            want = np.concatenate(want) if want else np.zeros((0,) + every.shape[1:], np.uint8)
            assert n.value == len(want)
            assert np.array_equal(path.canvases(n.value), want)
    path.close()


def test_device_descriptor_list_equals_host_compaction(ctx):
    """The planner's dense device descriptors (look-back prefix as the
    compaction scan) equal the host compaction of the per-frame slots,
    record for record, for a multi-camera shard."""
    import ctypes as C

    from paper_2404_09267_b200 import _native as N
    cams = [4, 5, 6]
    path = MC.MultiCameraPath(ctx, cams, 1920, 1080, 9, PROFILE, bandwidth_mbps=40.0,
                              trace_kw=dict(roi_proportion_mean=0.2))
    path.run_planes()
    desc = path.descriptors().copy()
    F, Z = len(cams) * 9, path.zones
    res = path.pipe.results(F, path.stream)
    patches = np.ctypeslib.as_array(C.cast(res["patches"], C.POINTER(C.c_uint8)),
                                    shape=(F * Z * 64,)).copy()
    out = np.zeros(F * Z, MC.DESC_DTYPE)
    n = C.c_int64()
    A.check(N.lib().tg_descriptors_compact(patches.ctypes.data, res["n_patches"].ctypes.data,
                                           np.ascontiguousarray(res["admitted"]).ctypes.data, Z,
                                           np.array(cams, np.int32).ctypes.data, len(cams), 9,
                                           out.ctypes.data, len(out), C.byref(n)))
    assert n.value == len(desc) > 0
    assert out[:n.value].tobytes() == desc.tobytes()
    assert list(np.unique(desc["camera"])) == cams
    path.close()


def test_nccl_single_rank_comm_matches_local_path(ctx):
    """With an NCCL communicator (one rank) the descriptor blocks go through
    ncclAllGather on the device; events and canvases equal the local path."""
    cams = [0, 1]
    local = MC.MultiCameraPath(ctx, cams, 1920, 1080, 8, PROFILE, bandwidth_mbps=40.0,
                               trace_kw=dict(roi_proportion_mean=0.15))
    _, ne, nc = local.step()
    ctx.stream_sync(local.stream)
    want_ev = [(e.fire_time_us, e.trigger, e.batch_size, e.patch_ids) for e in local.events()]
    want = local.canvases(nc)
    local.close()
    comm = A.Comm.nccl(ctx, A.Comm.unique_id(), 0, 1)
    path = MC.MultiCameraPath(ctx, cams, 1920, 1080, 8, PROFILE, bandwidth_mbps=40.0,
                              trace_kw=dict(roi_proportion_mean=0.15), comm=comm)
    assert path.d_blocks is not None
    got_n = path.run_pipelined(2)
    ctx.stream_sync(path.stream)
    assert got_n == nc
    assert [(e.fire_time_us, e.trigger, e.batch_size, e.patch_ids) for e in path.events()] == want_ev
    assert np.array_equal(path.canvases(nc), want)
    path.close()
    comm.close()


def test_descriptor_output_capacity_and_detach(ctx):
    """A run with more patches than the attached block holds latches
    TG_ERR_CAPACITY (the block keeps cap records); detaching stops the
    output; the camera table maps frames to (camera, frame)."""
    from paper_2404_09267_b200 import _native as N
    from tests._helpers import GpuRun
    run = GpuRun(ctx, 1920, 1080, 6, seed=11, keep_mask=False,
                 trace_kw=dict(roi_proportion_mean=0.3))
    run.run()
    total = int(run.res["n_patches"].sum())
    assert total > 4
    cap = total - 3
    blk = ctx.malloc(MC.block_bytes(total))
    cams = ctx.malloc(8)
    ctx.upload(cams, np.array([5, 9], np.int32))
    run.pipe.set_descriptor_output(blk, cap, cams, 3)  # frames 0-2: camera 5, 3-5: camera 9
    with pytest.raises(A.CapacityError, match="descriptor capacity exceeded"):
        run.run()
    got = ctx.download(blk, (MC.block_bytes(cap),), np.uint8)
    recs = MC.flatten_blocks(got.ctypes.data, 1, cap)
    assert len(recs) == cap
    assert list(recs["patch"]["patch_id"]) == list(range(cap))
    n0 = int(run.res["n_patches"][:3].sum())
    assert set(recs["camera"][:n0]) <= {5} and set(recs["camera"][n0:]) <= {9}
    assert list(recs["frame"][:n0]) == sorted(recs["frame"][:n0])
    run.pipe.set_descriptor_output(blk, total, cams, 3)
    run.run()
    got = ctx.download(blk, (MC.block_bytes(total),), np.uint8)  # kept alive while read
    recs = MC.flatten_blocks(got.ctypes.data, 1, total)
    assert len(recs) == total
    ctx.memset(blk, 0, MC.block_bytes(cap))
    run.pipe.set_descriptor_output(None)
    run.run()  # detached: the block is not written
    assert not ctx.download(blk, (MC.block_bytes(cap),), np.uint8).any()
    with pytest.raises(A.InvalidArgument):
        run.pipe.set_descriptor_output(blk + 4, 8)
    for p in (blk, cams):
        ctx.free(p)
    run.close()
    del N
