"""Multi-rank host logic of configs 3/4 on CPU (gloo, world size 2).

Each rank owns a contiguous block of cameras, builds its cameras' patch
descriptors (here from the oracle partition of the generator's rects, which
the device partition equals bit for bit -- test_gpu_parity), all-gathers them
as descriptor blocks through the C ABI's communicator with a host transport
(tg_comm_create_host; gloo moves the bytes) and checks that every rank holds
the global camera-major list (block layout, headers, flattening); then each
rank batches its shard with the SLO batcher and must reproduce the
reference simulator (tangram::run) run on exactly that shard's scenes.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from paper_2404_09267_b200 import multicam as MC

N_CAMS, N_FRAMES, W, H = 5, 16, 1920, 1080
PROFILE = [(1, 60.0, 3.0), (2, 85.0, 4.0), (4, 135.0, 6.0), (8, 235.0, 10.0)]


def scene(c):
    cfg = O.gen_cfg(seed=1000 + c, n_frames=N_FRAMES, fps=30.0, frame_width=W, frame_height=H,
                    roi_proportion_mean=0.15)
    return O.generate_trace(cfg)


def descriptors(cameras):
    recs = []
    for c in cameras:
        t_us, frames = scene(c)
        for f, rois in enumerate(frames):
            for p in O.partition(f, W, H, t_us[f], 1_000_000, 4, 4, rois, 1.5, 0):
                r = np.zeros(1, MC.DESC_DTYPE)[0]
                pp = r["patch"]
                pp["patch_id"] = p["patch_id"]
                pp["source_frame_id"] = p["source_frame_id"]
                pp["x"], pp["y"], pp["w"], pp["h"] = p["rect"]
                pp["generation_time_us"] = p["generation_time_us"]
                pp["slo_us"] = p["slo_us"]
                pp["deadline_us"] = p["deadline_us"]
                pp["size_bytes"] = p["size_bytes"]
                r["patch"] = pp
                r["camera"], r["frame"] = c, f
                r["admitted"] = int(p["rect"][2] <= 1024 and p["rect"][3] <= 1024)
                recs.append(r)
    return np.array(recs, MC.DESC_DTYPE)


def gloo_comm(rank, world):
    """api.Comm over a host transport: gloo all-gathers the byte strings."""
    import torch

    def allgather(data: bytes):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.numpy().tobytes() for p in parts]
    return A.Comm.host(rank, world, allgather)


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        mine = MC.shard_cameras(N_CAMS, world, rank)
        local = descriptors(mine)
        comm = gloo_comm(rank, world)
        per_rank = max(len(MC.shard_cameras(N_CAMS, world, r)) for r in range(world))
        glob = MC.allgather_descriptors(comm, local, per_rank * N_FRAMES * 16)
        full = descriptors(range(N_CAMS))
        same = (glob.tobytes() == full.tobytes())
        sched = A.SloScheduler(A.CanvasSpec(1024, 1024), A.LatencyProfile(1024, 1024, PROFILE),
                               A.max_canvases_per_batch(6.0, 2.0, 1.0))
        n_ev, arrival, _ = MC.schedule_descriptors(sched, local, mine, N_FRAMES, 40.0)
        evs = [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us, e.patch_ids)
               for e in sched._events(n_ev)]
        # the same shard scheduled from the all-gathered list: global ids
        # (sim.hpp:249-251), other shards' records skipped -- same decisions
        sched_g = A.SloScheduler(A.CanvasSpec(1024, 1024), A.LatencyProfile(1024, 1024, PROFILE),
                                 A.max_canvases_per_batch(6.0, 2.0, 1.0))
        n_g, _, _ = MC.schedule_descriptors(sched_g, glob, mine, N_FRAMES, 40.0)
        off = int((glob["camera"] < mine[0]).sum())
        evs_g = [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us,
                  [i - off for i in e.patch_ids]) for e in sched_g._events(n_g)]
        same = same and evs_g == evs
        # global cross-camera mode: every rank replays ONE batcher over all
        # cameras from the gathered list -- the reference's single scheduler
        sched_all = A.SloScheduler(A.CanvasSpec(1024, 1024),
                                   A.LatencyProfile(1024, 1024, PROFILE),
                                   A.max_canvases_per_batch(6.0, 2.0, 1.0))
        n_all, _, plan_all = MC.schedule_descriptors(sched_all, glob, range(N_CAMS), N_FRAMES, 40.0)
        evs_all = [(e.fire_time_us, e.trigger, e.batch_size, e.estimated_slack_us, e.patch_ids)
                   for e in sched_all._events(n_all)]
        ref = None
        if O.have_ref():
            r = O.run_tangram([scene(c) for c in mine], W, H, PROFILE, bandwidth_mbps=40.0)
            names = {0: "deadline_timer", 1: "infeasible_arrival", 2: "memory_cap"}
            ref = [(e["fire_time_us"], names[e["trigger"]], e["batch_size"], e["estimated_slack_us"],
                    e["patch_ids"]) for e in r["events"]]
            r = O.run_tangram([scene(c) for c in range(N_CAMS)], W, H, PROFILE, bandwidth_mbps=40.0)
            ref_all = [(e["fire_time_us"], names[e["trigger"]], e["batch_size"],
                        e["estimated_slack_us"], e["patch_ids"]) for e in r["events"]]
            same = same and evs_all == ref_all
            # infeasible-at-arrival flags of the admitted patches (sim.hpp:296-300)
            ref_inf = [f for f, a in zip(r["infeasible"], r["admitted"]) if a]
            same = same and [bool(x) for x in plan_all["infeasible"]] == [bool(x) for x in ref_inf]
        q.put((rank, mine, same, len(glob), evs, ref))
        comm.close()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, None, repr(e), 0, None, None))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_sharding_is_contiguous_and_complete():
    for world in (1, 2, 4, 8):
        owned = [MC.shard_cameras(64, world, r) for r in range(world)]
        assert sorted(c for o in owned for c in o) == list(range(64))
        for o in owned:
            assert o == list(range(o[0], o[-1] + 1)) and len(o) == 64 // world


def test_two_rank_descriptor_allgather_and_shard_batching():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, mine, same, n_glob, evs, ref in res:
        assert mine is not None, same
        assert same is True, (f"rank {rank}: gathered list, shard-from-gathered schedule or global "
                              "batching differs")
        assert n_glob == len(descriptors(range(N_CAMS)))
        assert evs, rank
        if ref is not None:
            assert evs == ref, f"rank {rank}: shard batching differs from the reference simulator"
    assert sorted(c for _, mine, *_ in res for c in mine) == list(range(N_CAMS))


def test_descriptor_blocks_round_trip():
    """Host blocks: header (count, cap) + records; flattening concatenates
    the valid records of every block and rejects corrupt headers."""
    import ctypes as C
    recs = descriptors([0, 1])
    a, b = recs[:7], recs[7:20]
    buf = np.concatenate([MC.descriptor_block(a, 32), MC.descriptor_block(b, 32)])
    assert buf.nbytes == 2 * MC.block_bytes(32) == 2 * 80 * 33
    got = MC.flatten_blocks(buf.ctypes.data, 2, 32)
    assert got.tobytes() == np.concatenate([a, b]).tobytes()
    assert len(MC.flatten_blocks(MC.descriptor_block(recs[:0], 4).ctypes.data, 1, 4)) == 0
    bad = MC.descriptor_block(a, 32)
    bad[:8].view(np.int64)[0] = 33
    with pytest.raises(A.InvalidArgument, match="holds 33 records"):
        MC.flatten_blocks(bad.ctypes.data, 1, 32)
    with pytest.raises(A.CapacityError):
        MC.flatten_blocks(buf.ctypes.data, 2, 32, out=np.zeros(10, MC.DESC_DTYPE))
    with pytest.raises(ValueError):
        MC.descriptor_block(recs, 4)
    del C


def test_host_comm_single_rank_and_failing_transport():
    comm = A.Comm.host(0, 1, lambda data: [data])
    recs = descriptors([3])
    assert MC.allgather_descriptors(comm, recs, len(recs)).tobytes() == recs.tobytes()
    assert comm.allgather_bytes(b"abc") == [b"abc"]
    comm.close()
    broken = A.Comm.host(0, 2, lambda data: [data])  # returns one part for two ranks
    with pytest.raises(A.TangramError, match="host transport failed"):
        broken.allgather_bytes(b"xy")
    broken.close()
    with pytest.raises(A.InvalidArgument):
        A.Comm.host(2, 2, lambda d: [d, d])
