"""Regenerates tests/golden/golden.json -- run in the authoring container.

Rect-level vectors come from the REFERENCE ITSELF (oracle/_ref, the
reference headers compiled as-is); pixel-stage vectors (absent from the
reference) come from the frozen C restatement, with the rect stages inside
that path again executed by the reference.  The committed JSON is what the
CPU tests check the oracle port against, so the port is pinned even on a box
where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

LIB = "ref"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rect_vectors():
    g = {}
    # partition_test.cpp:27-126 and SPEC.md:104-125 KATs, recomputed by the reference.
    g["zones"] = {
        "100x100_2x2": O.make_zones(100, 100, 2, 2, LIB),
        "101x100_2x2": O.make_zones(101, 100, 2, 2, LIB),
        "3840x2160_4x4": O.make_zones(3840, 2160, 4, 4, LIB),
        "1920x1080_6x6": O.make_zones(1920, 1080, 6, 6, LIB),
    }
    kat = [
        dict(frame=(7, 100, 100, 250000, 500000), grid=(2, 2), rois=[(30, 10, 30, 20), (5, 5, 10, 10)], bpp=1.5, first=40),
        dict(frame=(0, 100, 100, 0, 500000), grid=(2, 2), rois=[(10, 10, 10, 10), (60, 10, 10, 10), (10, 60, 10, 10)], bpp=1.0, first=0),
        dict(frame=(0, 100, 100, 0, 500000), grid=(2, 2), rois=[(40, 10, 20, 10)], bpp=1.0, first=0),
        dict(frame=(0, 100, 100, 0, 500000), grid=(2, 2), rois=[(40, 40, 20, 20)], bpp=1.5, first=0),
        dict(frame=(0, 97, 53, 0, 500000), grid=(3, 2), rois=[(0, 0, 97, 53), (96, 52, 1, 1)], bpp=1.0, first=0),
        dict(frame=(0, 100, 100, 0, 500000), grid=(2, 2), rois=[], bpp=1.5, first=0),
    ]
    for k in kat:
        fid, w, h, gen, slo = k["frame"]
        k["patches"] = O.partition(fid, w, h, gen, slo, *k["grid"], k["rois"], k["bpp"], k["first"], lib=LIB)
    g["partition_kats"] = kat
    errs = {}
    for name, args in {"outside": (0, 100, 100, 0, 1, 2, 2, [(200, 200, 10, 10)], 1.5),
                       "finer": (0, 3, 3, 0, 1, 4, 4, [], 1.5)}.items():
        try:
            O.partition(*args, lib=LIB)
        except O.OracleError as e:
            errs[name] = str(e)
    g["partition_errors"] = errs

    # stitch_test.cpp:42-193 KATs.
    sk = []
    for q, cw, ch in [([(0, 50, 100), (1, 50, 100)], 100, 100), ([(0, 60, 60), (1, 50, 50)], 100, 100),
                      ([(0, 100, 100)], 100, 100), ([(0, 60, 60), (1, 40, 40)], 100, 100),
                      ([(0, 60, 60), (1, 30, 30)], 100, 100), ([], 100, 100)]:
        pl, nc, fr = O.stitch_all(q, cw, ch, LIB)
        sk.append(dict(queue=q, canvas=(cw, ch), placements=pl, n_canvases=nc, free=fr))
    g["stitch_kats"] = sk
    try:
        O.stitch_all([(0, 101, 10)], 100, 100, LIB)
    except O.OracleError as e:
        g["stitch_error"] = str(e)

    # acceptance_test.cpp:48-101 (C01) generator: derive_seed(2026,"packing"),
    # n in [1,24], dims in [16,1024]; first 400 sets with full outputs.
    rng = O.Rng(O.derive_seed(2026, "packing", LIB))
    sets = []
    for _ in range(400):
        n = rng.uniform_int(1, 24)
        q = [(i, rng.uniform_int(16, 1024), rng.uniform_int(16, 1024)) for i in range(n)]
        pl, nc, fr = O.stitch_all(q, 1024, 1024, LIB)
        sets.append(dict(queue=q, placements=pl, n_canvases=nc, free=fr))
    g["c01_sets"] = sets

    # Generator (trace.hpp:184-231) for the BASELINE configs' cameras.
    traces = {}
    for name, kw in {
        "cfg1_seed1000": dict(seed=1000, n_frames=30, fps=30.0),
        "cfg2_seed1000": dict(seed=1000, n_frames=300, fps=30.0, frame_width=3840, frame_height=2160),
        "default_seed7": dict(seed=7, n_frames=60),
        "dense_seed1001": dict(seed=1001, n_frames=40, fps=30.0, frame_width=3840, frame_height=2160,
                               roi_proportion_mean=0.59, roi_max_dim=1024, roi_count_max=24),
    }.items():
        cfg = O.gen_cfg(**kw)
        t_us, frames = O.generate_trace(cfg, LIB)
        # Reference partition of the generator's own rects (sim.hpp:243-272, 4x4 grid).
        parts, first = [], 0
        for i, rois in enumerate(frames):
            p = O.partition(i, cfg.frame_width, cfg.frame_height, t_us[i], 1_000_000, 4, 4, rois, 1.5,
                            first, lib=LIB)
            first += len(p)
            parts.append([(q["patch_id"], *q["rect"], q["size_bytes"]) for q in p])
        traces[name] = dict(cfg=kw, t_us=t_us, rois=frames, patches=parts)
    g["traces"] = traces
    return g


def pixel_vectors():
    """Frozen pixel spec vectors (parity unpinned by the reference)."""
    out = {}
    for name, (W, H, n, seed, radius) in {
        "cfg1_1080p_4f": (1920, 1080, 4, 1000, 2),
        "small_320x192_5f_r0": (320, 192, 5, 77, 0),
        "small_96x64_6f_r3": (96, 64, 6, 5, 3),
    }.items():
        cfg = O.gen_cfg(seed=seed, n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                        roi_max_dim=min(480, W, H))
        t_us, frames = O.generate_trace(cfg, LIB)
        ps = O.derive_seed(seed, "pixels", LIB)
        fr = [O.synth_frame(W, H, ps, -1, [])] + [O.synth_frame(W, H, ps, i, frames[i]) for i in range(n)]
        params = dict(width=W, height=H, pitch=W * 3, threshold=25, radius=radius, zones_x=4, zones_y=4,
                      canvas_w=1024, canvas_h=1024, bytes_per_pixel=1.5, slo_us=1_000_000, max_rois=1024,
                      threads=4)
        res = O.process_frames(params, fr[1:], fr[:-1], list(range(n)), t_us, want_cells=True, lib=LIB)
        masks = [O.mask(fr[i + 1], fr[i], W, H, 25, radius) for i in range(n)]
        out[name] = dict(
            W=W, H=H, n=n, seed=seed, radius=radius,
            frame_sha=[sha(f) for f in fr],
            mask_sha=[sha(m) for m in masks],
            cells_sha=[sha(c) for c in res["cells"]],
            rois=[res["rois"][i, :res["n_rois"][i]].tolist() for i in range(n)],
            patches=[[(q["patch_id"], *q["rect"], q["size_bytes"]) for q in p] for p in res["patch_list"]],
            placements=res["placement_list"],
            n_canvases=res["n_canvases"].tolist(),
            canvas_sha=[sha(res["canvases"][k]) for k in range(res["total_canvases"])],
        )
    return out


def main():
    if not O.have_ref():
        O.build()
    g = {"generator": "tests/golden/make_golden.py", "rect": rect_vectors(), "pixel": pixel_vectors()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
