"""Global cross-camera mode on the device: 2 or 3 ranks --
processes sharing this one GPU, gloo for the host exchange -- each run K1-K4 on
their own cameras, all-gather the descriptors, replay ONE batcher over every
camera and write the canvases of their share of the invoke events, reading
the other ranks' frames through CUDA IPC.

Checks: all ranks take identical decisions, equal to the reference
simulator (tangram::run) over all cameras on the GPU-extracted RoIs; every
canvas byte of every event equals a host fill from the frames; the ranks'
event shares partition the events.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_CAMS, N_FRAMES, W, H, BW = 5, 8, 1920, 1080, 40.0
PROFILE = [(1, 60.0, 3.0), (2, 85.0, 4.0), (4, 135.0, 6.0), (8, 235.0, 10.0)]


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        from paper_2404_09267_b200 import api as A
        from paper_2404_09267_b200 import multicam as MC
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ctx = A.Context(0)
        import torch

        def allgather(data: bytes):  # host transport: NCCL refuses two ranks on one GPU
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return [p.numpy().tobytes() for p in parts]
        comm = A.Comm.host(rank, world, allgather)
        path = MC.GlobalCameraPath(ctx, N_CAMS, comm, W, H, N_FRAMES, PROFILE,
                                   bandwidth_mbps=BW, trace_kw=dict(roi_proportion_mean=0.15))
        desc, n_events, n_canv = path.step()
        ctx.stream_sync(path.stream)
        events = path.events()
        # RoIs of my cameras, shared so every rank can rebuild the global scene list
        mine = {c: path.camera_results(k) for k, c in enumerate(path.cameras)}
        rois = {c: [[tuple(r) for r in res["rois"][f, :res["n_rois"][f]].tolist()]
                    for f in range(N_FRAMES)] for c, res in mine.items()}
        every = [None] * world
        dist.all_gather_object(every, rois)
        all_rois = {c: r for part in every for c, r in part.items()}
        # every camera's frames, read through the global (IPC) frame table
        fb = 3 * W * H
        frames = {c: [ctx.download(path.frame_base[c] + s * fb, (H, 3 * W), np.uint8)
                      for s in range(N_FRAMES + 1)] for c in path.all_cameras}
        plan = path._last
        by_id = {int(p["patch_id"]): (int(s), p) for p, s in zip(plan["patches"], plan["src"])}
        got = path.canvases(n_canv)
        k, bad = 0, []
        for ei, e in enumerate(events):
            if ei % world != rank:
                continue
            for cv in e.stitch.canvases:
                want = np.zeros((1024, 1024 * 3), np.uint8)
                for pl in cv.placements:
                    src, p = by_id[pl.patch_id]
                    cam, slot = divmod(src, N_FRAMES + 1)
                    fr = frames[cam][slot]
                    x, y, w, h = pl.position.x, pl.position.y, pl.position.w, pl.position.h
                    want[y:y + h, 3 * x:3 * (x + w)] = \
                        fr[p["y"]:p["y"] + h, 3 * p["x"]:3 * (p["x"] + w)]
                if not np.array_equal(got[k], want):
                    bad.append((ei, k))
                k += 1
        evs = [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us, e.patch_ids)
               for e in events]
        t_us = {c: path.t_us[path.cameras.index(c)] for c in path.cameras}
        every_t = [None] * world
        dist.all_gather_object(every_t, t_us)
        all_t = {c: t for part in every_t for c, t in part.items()}
        scenes = [(all_t[c], all_rois[c]) for c in range(N_CAMS)]
        q.put((rank, evs, scenes, k == n_canv, bad, n_canv))
        dist.barrier()
        path.close()
        comm.close()
        ctx.close()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        import traceback
        q.put((rank, None, traceback.format_exc(), False, [repr(e)], 0))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_global_cross_camera_mode_ranks_on_one_gpu(world):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    for rank, evs, scenes, counted, bad, n_canv in res:
        assert evs is not None, scenes
        assert counted and not bad, (rank, bad)
        assert n_canv > 0
    for r in res[1:]:
        assert r[1] == res[0][1], "ranks took different batching decisions"
        assert r[2] == res[0][2]
    evs = res[0][1]
    assert sum(r[5] for r in res) == sum(e[2] for e in evs)
    if O.have_ref():
        ref = O.run_tangram(res[0][2], W, H, PROFILE, bandwidth_mbps=BW)
        names = {0: "deadline_timer", 1: "infeasible_arrival", 2: "memory_cap"}
        assert evs == [(e["fire_time_us"], names[e["trigger"]], e["batch_size"],
                        e["estimated_slack_us"], e["patch_ids"]) for e in ref["events"]]
