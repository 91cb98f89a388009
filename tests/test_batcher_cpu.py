"""The SLO batcher (Alg. 2 invoker) against the reference scheduler.

The batcher is host code over descriptors (it never touches pixels), so
these run without a GPU.  Checks, all exact:
* the reference's own unit-test KATs (scheduler_test.cpp:56-151);
* random arrival streams driven event by event against the reference
  SloScheduler compiled as-is (oracle/_ref), comparing every event's fire
  time, trigger, batch size, slack, patch ids, placements and free lists;
* multi-camera streams through the reference's whole simulator
  (tangram::run, tangram policy): admission, per-link arrival times
  (transmission_schedule) and every invoke in its event log.
"""
import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A

need_ref = pytest.mark.skipif(not O.have_ref(), reason="reference build (oracle/_ref) absent")

TEST_PROFILE = [(1, 100.0, 10.0), (2, 170.0, 10.0)]  # scheduler_test.cpp:33-35


def full_patch(pid, gen, slo):
    return A.PatchMeta(pid, pid, A.Rect(0, 0, 100, 100), gen, slo, gen + slo, 15000)


def sched(max_canvases=2, profile=TEST_PROFILE, canvas=(100, 100)):
    return A.SloScheduler(A.CanvasSpec(*canvas), A.LatencyProfile(*canvas, profile), max_canvases)


def test_single_arrival_arms_deadline_timer():
    s = sched()
    assert s.on_patch_arrival(full_patch(1, 0, 500_000), 0) == []
    assert not s.idle()
    assert s.earliest_deadline_us() == 500_000 and s.remaining_time_us() == 370_000
    t = s.pending_timer()
    assert t.fire_at_us == 370_000
    ev = s.on_timer(370_000, t.epoch)
    assert (ev.fire_time_us, ev.batch_size, ev.patch_ids, ev.estimated_slack_us, ev.trigger) == \
        (370_000, 1, [1], 130_000, "deadline_timer")
    assert s.idle() and s.pending_timer() is None


def test_second_arrival_rearms_with_batch_slack():
    s = sched()
    s.on_patch_arrival(full_patch(1, 0, 500_000), 0)
    stale = s.pending_timer().epoch
    assert s.on_patch_arrival(full_patch(2, 100_000, 500_000), 100_000) == []
    assert s.queue_size() == 2 and s.current_canvas_count() == 2
    assert [p.patch_id for p in s.queue()] == [1, 2] and s.current_stitch().canvas_count() == 2
    assert s.remaining_time_us() == 300_000 and s.pending_timer().fire_at_us == 300_000
    assert s.on_timer(370_000, stale) is None
    ev = s.on_timer(300_000, s.pending_timer().epoch)
    assert ev.batch_size == 2 and ev.patch_ids == [1, 2] and ev.estimated_slack_us == 200_000


def test_memory_cap_flushes_previous_batch():
    s = sched()
    s.on_patch_arrival(full_patch(1, 0, 500_000), 0)
    s.on_patch_arrival(full_patch(2, 100_000, 500_000), 100_000)
    evs = s.on_patch_arrival(full_patch(3, 250_000, 500_000), 250_000)
    assert len(evs) == 1
    e = evs[0]
    assert (e.trigger, e.fire_time_us, e.batch_size, e.patch_ids, e.estimated_slack_us) == \
        ("memory_cap", 250_000, 2, [1, 2], 200_000)


def test_constructor_validation_and_profile():
    with pytest.raises(A.InvalidArgument):
        A.SloScheduler(A.CanvasSpec(100, 100), A.LatencyProfile(100, 100, TEST_PROFILE), 0)
    with pytest.raises(A.InvalidArgument, match="latency profile has no entries"):
        A.LatencyProfile(100, 100, [])
    with pytest.raises(A.InvalidArgument, match="duplicate profile entry"):
        A.LatencyProfile(100, 100, [(1, 10.0, 1.0), (1, 11.0, 1.0)])
    p = A.LatencyProfile(100, 100, TEST_PROFILE)
    assert [p.slack_us(k) for k in (1, 2, 3)] == [130_000, 200_000, 270_000]
    assert A.max_canvases_per_batch(6.0, 2.0, 1.0) == 4
    with pytest.raises(A.InvalidArgument, match="cannot fit one canvas"):
        A.max_canvases_per_batch(2.5, 2.0, 1.0)


def random_patches(seed, n):
    """scheduler_test.cpp:236-255."""
    rng = O.Rng(seed)
    out, t = [], 0
    for i in range(n):
        t += rng.uniform_int(0, 120_000)
        w, h = rng.uniform_int(10, 100), rng.uniform_int(10, 100)
        slo = rng.uniform_int(125_000, 2_000_000)
        out.append(A.PatchMeta(i + 1, i, A.Rect(0, 0, w, h), t, slo, t + slo, w * h))
    return out


def drive(s, patches, ref=None):
    """scheduler_test.cpp:216-233: timers due at or before each generation
    time fire first; every call is mirrored on the reference scheduler."""
    ours, theirs = [], []

    def d(p):
        return dict(patch_id=p.patch_id, source_frame_id=p.source_frame_id,
                    rect=(p.rect.x, p.rect.y, p.rect.w, p.rect.h),
                    generation_time_us=p.generation_time_us, slo_us=p.slo_us,
                    deadline_us=p.deadline_us, size_bytes=p.size_bytes)

    def fire_due(limit):
        while s.pending_timer() is not None and (limit is None or s.pending_timer().fire_at_us <= limit):
            t = s.pending_timer()
            if ref is not None:
                assert ref.pending_timer() == (t.fire_at_us, t.epoch)
                r = ref.on_timer(t.fire_at_us, t.epoch)
                if r:
                    theirs.append(r)
            e = s.on_timer(t.fire_at_us, t.epoch)
            if e:
                ours.append(e)

    for p in patches:
        fire_due(p.generation_time_us)
        ours.extend(s.on_patch_arrival(p, p.generation_time_us))
        if ref is not None:
            theirs.extend(ref.on_patch_arrival(d(p), p.generation_time_us))
    fire_due(None)
    return ours, theirs


def event_tuple(e):
    pl = [(p.patch_id, p.canvas_index, p.position.x, p.position.y, p.position.w, p.position.h)
          for c in e.stitch.canvases for p in c.placements]
    fr = [(ci, r.x, r.y, r.w, r.h) for ci, c in enumerate(e.stitch.canvases) for r in c.free_rects]
    trig = {"deadline_timer": 0, "infeasible_arrival": 1, "memory_cap": 2}[e.trigger]
    return (e.fire_time_us, trig, e.batch_size, e.estimated_slack_us, e.patch_ids, pl, fr)


def ref_tuple(e):
    return (e["fire_time_us"], e["trigger"], e["batch_size"], e["estimated_slack_us"],
            e["patch_ids"], e["placements"], e["free"])


def test_every_admitted_patch_fires_exactly_once():
    """scheduler_test.cpp:257-290 invariants."""
    prof = A.LatencyProfile(100, 100, TEST_PROFILE)
    for seed in range(1, 21):
        s = sched(3)
        patches = random_patches(seed, 200)
        events, _ = drive(s, patches)
        deadline = {p.patch_id: p.deadline_us for p in patches}
        seen, last = set(), 0
        for e in events:
            assert e.fire_time_us >= last
            last = e.fire_time_us
            assert 1 <= e.batch_size <= 3
            assert e.estimated_slack_us == prof.slack_us(e.batch_size)
            for pid in e.patch_ids:
                assert pid not in seen
                seen.add(pid)
            if e.trigger == "deadline_timer":
                assert e.fire_time_us == min(deadline[i] for i in e.patch_ids) - e.estimated_slack_us
        assert len(seen) == len(patches) and s.idle()


@need_ref
@pytest.mark.parametrize("canvas,max_canvases,profile", [
    ((100, 100), 3, TEST_PROFILE),
    ((256, 256), 2, [(1, 40.0, 4.0), (2, 60.0, 5.0), (4, 95.0, 8.0)]),
    ((1024, 1024), 8, [(1, 60.0, 3.0), (2, 85.0, 4.0), (4, 135.0, 6.0), (8, 235.0, 10.0)]),
])
def test_random_streams_match_reference_scheduler(canvas, max_canvases, profile):
    for seed in range(1, 31):
        s = sched(max_canvases, profile, canvas)
        ref = O.RefScheduler(canvas[0], canvas[1], profile, max_canvases)
        patches = random_patches(seed * 7 + canvas[0], 150)
        ours, theirs = drive(s, patches, ref)
        assert [event_tuple(e) for e in ours] == [ref_tuple(e) for e in theirs], seed


def scenes_for(n_cams, n_frames, W, H, **kw):
    out = []
    for c in range(n_cams):
        cfg = O.gen_cfg(seed=1000 + c, n_frames=n_frames, fps=30.0, frame_width=W, frame_height=H, **kw)
        out.append(O.generate_trace(cfg))
    return out


def our_run(scenes, W, H, profile, bandwidth, zones=(4, 4), canvas=(1024, 1024), gpu_mem=6.0,
            model=2.0, slo=1_000_000):
    """The device-side pipeline's host half for configs 3/4: partition (here
    the oracle's, bit-identical to the device's), admission (sim.hpp:262),
    per-camera link arrivals, then the batcher's reference event loop."""
    first = 0
    admitted_all, arrival_of = [], {}
    order_patches, order_arrivals = [], []
    for t_us, frames in scenes:
        adm = []
        for i, rois in enumerate(frames):
            patches = O.partition(i, W, H, t_us[i], slo, zones[0], zones[1], rois, 1.5, first)
            first += len(patches)
            for p in patches:
                ok = p["rect"][2] <= canvas[0] and p["rect"][3] <= canvas[1]
                admitted_all.append(ok)
                if ok:
                    adm.append(A.PatchMeta(p["patch_id"], p["source_frame_id"], A.Rect(*p["rect"]),
                                           p["generation_time_us"], p["slo_us"], p["deadline_us"],
                                           p["size_bytes"]))
        arr = A.transmission_schedule(adm, bandwidth)
        for p, a in zip(adm, arr):
            arrival_of[p.patch_id] = a
        order_patches += adm
        order_arrivals += arr
    s = A.SloScheduler(A.CanvasSpec(*canvas), A.LatencyProfile(*canvas, profile),
                       A.max_canvases_per_batch(gpu_mem, model, 1.0))
    s.enable_log("tangram")
    events = s.replay(order_patches, order_arrivals)
    our_run.log = s.take_log()
    return admitted_all, arrival_of, events


SIM_PROFILE = [(1, 60.0, 3.0), (2, 85.0, 4.0), (4, 135.0, 6.0), (8, 235.0, 10.0)]


@need_ref
@pytest.mark.parametrize("n_cams,W,H,bw,kw", [
    (1, 1920, 1080, 80.0, {}),
    (5, 3840, 2160, 80.0, dict(roi_max_dim=480)),            # config 3 geometry
    (5, 3840, 2160, 20.0, dict(roi_max_dim=1024, roi_proportion_mean=0.3)),
    (8, 1920, 1080, 40.0, dict(roi_proportion_mean=0.2)),
])
def test_multi_camera_stream_matches_reference_simulator(n_cams, W, H, bw, kw):
    scenes = scenes_for(n_cams, 24, W, H, **kw)
    ref = O.run_tangram(scenes, W, H, SIM_PROFILE, bandwidth_mbps=bw)
    admitted, arrival_of, events = our_run(scenes, W, H, SIM_PROFILE, bw)
    assert admitted == [bool(a) for a in ref["admitted"]]
    for pid, a in arrival_of.items():
        assert ref["arrival_us"][pid] == a
    ours = [(e.fire_time_us, {"deadline_timer": 0, "infeasible_arrival": 1, "memory_cap": 2}[e.trigger],
             e.batch_size, e.estimated_slack_us, e.patch_ids) for e in events]
    theirs = [(e["fire_time_us"], e["trigger"], e["batch_size"], e["estimated_slack_us"],
               e["patch_ids"]) for e in ref["events"]]
    assert ours == theirs
    assert len(ours) > 0
    # the whole event log (arrival / repack / invoke / timer_set lines),
    # byte for byte (scheduler_test.cpp:302-320 replays it the same way)
    assert our_run.log == ref["log"]


@need_ref
@pytest.mark.parametrize("per_camera_link", [True, False])
def test_replay_links_matches_reference_simulator(per_camera_link):
    """tg_batcher_replay_links (the link model of sim.hpp:274-290 + the event
    loop in one call): per-camera FIFO uplinks and the single shared link
    sorted by (generation time, patch id), against tangram::run."""
    W, H, bw = 1920, 1080, 30.0
    scenes = scenes_for(4, 20, W, H, roi_proportion_mean=0.2)
    ref = O.run_tangram(scenes, W, H, SIM_PROFILE, bandwidth_mbps=bw,
                        per_scene_link=per_camera_link)
    first, cams = 0, []
    for t_us, frames in scenes:
        adm = []
        for i, rois in enumerate(frames):
            patches = O.partition(i, W, H, t_us[i], 1_000_000, 4, 4, rois, 1.5, first)
            first += len(patches)
            adm += [A.PatchMeta(p["patch_id"], p["source_frame_id"], A.Rect(*p["rect"]),
                                p["generation_time_us"], p["slo_us"], p["deadline_us"], p["size_bytes"])
                    for p in patches if p["rect"][2] <= 1024 and p["rect"][3] <= 1024]
        cams.append(adm)
    s = A.SloScheduler(A.CanvasSpec(1024, 1024), A.LatencyProfile(1024, 1024, SIM_PROFILE),
                       A.max_canvases_per_batch(6.0, 2.0, 1.0))
    s.enable_log("tangram")
    events, arrivals = s.replay_links(cams, bw, per_camera_link)
    flat = [p for cam in cams for p in cam]
    for p, a in zip(flat, arrivals):
        assert ref["arrival_us"][p.patch_id] == a
    ours = [(e.fire_time_us, {"deadline_timer": 0, "infeasible_arrival": 1, "memory_cap": 2}[e.trigger],
             e.batch_size, e.estimated_slack_us, e.patch_ids) for e in events]
    theirs = [(e["fire_time_us"], e["trigger"], e["batch_size"], e["estimated_slack_us"],
               e["patch_ids"]) for e in ref["events"]]
    assert ours == theirs and len(ours) > 0
    assert s.take_log() == ref["log"]


def test_descriptor_compaction_layout():
    """tg_descriptors_compact: pipeline slots [F][Z] -> camera-major records."""
    import ctypes as C

    import numpy as np

    from paper_2404_09267_b200 import _native as N
    from paper_2404_09267_b200 import multicam as MC
    rng = np.random.default_rng(5)
    cams, n, Z = np.array([3, 7, 9], np.int32), 4, 16
    F = len(cams) * n
    pat = np.zeros(F * Z, MC.PATCH_DTYPE)
    pat["patch_id"] = np.arange(F * Z)
    pat["w"] = rng.integers(1, 2000, F * Z)
    adm = rng.integers(0, 2, F * Z).astype(np.uint8)
    cnt = rng.integers(0, Z + 1, F).astype(np.int32)
    out = np.zeros(F * Z, MC.DESC_DTYPE)
    k = C.c_int64()
    A.check(N.lib().tg_descriptors_compact(pat.ctypes.data, cnt.ctypes.data, adm.ctypes.data, Z,
                                           cams.ctypes.data, len(cams), n, out.ctypes.data,
                                           len(out), C.byref(k)))
    valid = (np.arange(Z)[None, :] < cnt[:, None]).reshape(-1)
    assert k.value == int(valid.sum())
    got = out[:k.value]
    assert np.array_equal(got["patch"], pat[valid])
    assert np.array_equal(got["admitted"], adm[valid].astype(np.int32))
    assert np.array_equal(got["camera"], np.repeat(cams, n * Z)[valid])
    assert np.array_equal(got["frame"], np.tile(np.repeat(np.arange(n), Z), len(cams))[valid])
    with pytest.raises(A.CapacityError):
        A.check(N.lib().tg_descriptors_compact(pat.ctypes.data, cnt.ctypes.data, adm.ctypes.data,
                                               Z, cams.ctypes.data, len(cams), n, out.ctypes.data,
                                               max(0, k.value - 1), C.byref(k)))


def test_infeasible_arrival_flushes_then_requeues():
    """scheduler_test.cpp:133-162."""
    s = sched(4)
    a = full_patch(1, 0, 500_000)
    a.rect = A.Rect(0, 0, 50, 100)
    b = full_patch(2, 200_000, 260_000)
    b.rect = A.Rect(50, 0, 50, 100)
    assert s.on_patch_arrival(a, 0) == []
    assert s.on_patch_arrival(b, 200_000) == []
    assert s.current_canvas_count() == 1 and s.remaining_time_us() == 330_000
    c = full_patch(3, 340_000, 140_000)
    evs = s.on_patch_arrival(c, 340_000)
    assert len(evs) == 1
    assert (evs[0].trigger, evs[0].patch_ids, evs[0].batch_size) == ("infeasible_arrival", [1, 2], 1)
    assert s.queue_size() == 1 and s.remaining_time_us() == 350_000
    assert s.pending_timer().fire_at_us == 350_000


def test_solo_infeasible_patch_dispatches_immediately():
    """scheduler_test.cpp:164-177: SLO 120 ms < slack(1) = 130 ms."""
    s = sched(2)
    evs = s.on_patch_arrival(full_patch(1, 0, 120_000), 0)
    assert [(e.trigger, e.fire_time_us, e.batch_size, e.patch_ids) for e in evs] == \
        [("infeasible_arrival", 0, 1, [1])]
    assert s.idle() and s.pending_timer() is None


def test_flush_and_solo_dispatch_in_one_arrival():
    """scheduler_test.cpp:179-195."""
    s = sched(2)
    s.on_patch_arrival(full_patch(1, 0, 500_000), 0)
    evs = s.on_patch_arrival(full_patch(2, 300_000, 120_000), 300_000)
    assert [(e.trigger, e.patch_ids, e.fire_time_us) for e in evs] == \
        [("infeasible_arrival", [1], 300_000), ("infeasible_arrival", [2], 300_000)]
    assert s.idle()


def test_zero_remaining_time_still_feasible():
    """scheduler_test.cpp:197-209: deadline == slack(1) -> timer at now."""
    s = sched(2)
    assert s.on_patch_arrival(full_patch(1, 0, 130_000), 0) == []
    t = s.pending_timer()
    assert t is not None and t.fire_at_us == 0
    ev = s.on_timer(0, t.epoch)
    assert ev is not None and ev.trigger == "deadline_timer"


def test_timer_after_reset_is_ignored():
    """scheduler_test.cpp:211-219."""
    s = sched(2)
    s.on_patch_arrival(full_patch(1, 0, 500_000), 0)
    epoch = s.pending_timer().epoch
    assert s.on_timer(370_000, epoch) is not None
    assert s.on_timer(370_000, epoch) is None


def test_transmission_known_answers():
    """trace_test.cpp:243-275: 1 MB at 80 Mbps = 100 ms; FIFO link."""
    def sized(pid, gen, nbytes):
        return A.PatchMeta(pid, pid, A.Rect(0, 0, 1, 1), gen, 1_000_000, gen + 1_000_000, nbytes)

    assert A.transmission_schedule([sized(0, 0, 1_000_000)], 80.0) == [100_000]
    assert A.transmission_schedule([sized(0, 0, 2_000_000)], 80.0) == [200_000]
    assert A.transmission_schedule([sized(0, 0, 0)], 80.0) == [0]
    with pytest.raises(A.InvalidArgument):
        A.transmission_schedule([sized(0, 0, 100)], 0.0)
    assert A.transmission_schedule([sized(0, 0, 1_000_000), sized(1, 0, 1_000_000),
                                    sized(2, 150_000, 1_000_000)], 80.0) == \
        [100_000, 200_000, 300_000]
    assert A.transmission_schedule([sized(0, 40_000, 250_000)], 80.0) == [65_000]


def test_schedule_descriptors_edge_cases():
    """tg_batcher_schedule: empty input, cameras without patches, other
    shards' records (skipped, ids still consumed), out-of-order cameras."""
    import numpy as np

    from paper_2404_09267_b200 import multicam as MC

    def recs(spec):
        out = np.zeros(len(spec), MC.DESC_DTYPE)
        for i, (cam, frame, w) in enumerate(spec):
            p = out[i]["patch"]
            p["x"], p["y"], p["w"], p["h"] = 0, 0, w, 100
            p["generation_time_us"] = frame * 33_333
            p["slo_us"] = 1_000_000
            p["deadline_us"] = frame * 33_333 + 1_000_000
            p["size_bytes"] = w * 150
            out[i]["patch"] = p
            out[i]["camera"], out[i]["frame"], out[i]["admitted"] = cam, frame, int(w <= 1024)
        return out

    def mk():
        return A.SloScheduler(A.CanvasSpec(1024, 1024), A.LatencyProfile(1024, 1024, SIM_PROFILE), 8)

    n_ev, arr, plan = MC.schedule_descriptors(mk(), recs([]), [0, 1], 4, 80.0)
    assert n_ev == 0 and len(arr) == 0 and len(plan["patches"]) == 0
    # camera 1 has no patches; camera 3 belongs to another shard; one oversize patch
    d = recs([(0, 0, 100), (0, 1, 2000), (1 + 2, 0, 50), (2, 2, 300)])
    n_ev, arr, plan = MC.schedule_descriptors(mk(), d, [0, 1, 2], 4, 80.0)
    assert [int(p["patch_id"]) for p in plan["patches"]] == [0, 3]  # ids over all records
    assert list(plan["src"]) == [0 * 5 + 0 + 1, 2 * 5 + 2 + 1]      # slot * (n + 1) + frame + 1
    assert n_ev >= 1 and len(arr) == 2
    with pytest.raises(A.InvalidArgument, match="out of the camera order"):
        MC.schedule_descriptors(mk(), recs([(2, 0, 100), (0, 0, 100)]), [0, 2], 4, 80.0)
    with pytest.raises(A.InvalidArgument, match="frame 9 out of range"):
        MC.schedule_descriptors(mk(), recs([(0, 9, 100)]), [0], 4, 80.0)


def test_batcher_beyond_65535_canvases():
    """The host best-fit key covers any canvas count: the winner sits on
    canvas 65540 (see tests/test_gpu_parity.py::wide_key_queue)."""
    dims = [(60, 60)] + [(100, 100)] * 65539 + [(61, 61), (39, 39)]
    patches = [A.PatchMeta(i, i, A.Rect(0, 0, w, h), 0, 10**12, 10**12, w * h)
               for i, (w, h) in enumerate(dims)]
    s = sched(max_canvases=70000, profile=[(1, 1.0, 0.0), (2, 1.0, 0.0)])
    evs = s.replay(patches, [0] * len(patches))
    assert len(evs) == 1 and evs[0].batch_size == 65541
    last = evs[0].stitch.placement_index[len(dims) - 1]
    assert (last.canvas_index, last.position) == (65540, A.Rect(61, 0, 39, 39))
