"""Shared helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2404_09267_b200 import api as A


def oracle_params(W, H, radius=2, threshold=25, zones=(4, 4), canvas=(1024, 1024), max_rois=1024,
                  threads=8, pitch=None):
    return dict(width=W, height=H, pitch=pitch or 3 * W, threshold=threshold, radius=radius,
                zones_x=zones[0], zones_y=zones[1], canvas_w=canvas[0], canvas_h=canvas[1],
                bytes_per_pixel=1.5, slo_us=1_000_000, max_rois=max_rois, threads=threads)


class GpuRun:
    """Synthesizes a camera on the device, runs the pipeline, keeps results."""

    def __init__(self, ctx, W, H, n, seed=1000, radius=2, threshold=25, zones=(4, 4),
                 canvas=(1024, 1024), max_rois=1024, keep_mask=True, trace_kw=None,
                 rects=None, max_canvases=None, first_patch_id=0, pitch=None):
        self.ctx, self.W, self.H, self.n = ctx, W, H, n
        trace_kw = dict(trace_kw or {})
        if rects is None:
            self.t_us, frames = A.generate_trace(n_frames=n, fps=30.0, frame_width=W, frame_height=H,
                                                 seed=seed, **trace_kw)
        else:
            frames = [[A.Rect(*r) for r in fr] for fr in rects]
            self.t_us = [int(round(i * 1e6 / 30.0)) for i in range(n)]
        self.rects = frames
        self.ring = A.FrameRing(ctx, W, H, n, pitch=pitch)
        self.pixel_seed = A.derive_seed(seed, "pixels")
        self.ring.synthesize(self.pixel_seed, frames)
        self.max_canvases = max_canvases if max_canvases is not None else n * zones[0] * zones[1]
        self.pipe = A.Pipeline(ctx, W, H, dilate_radius=radius, threshold=threshold, zones=zones,
                               canvas=canvas, max_rois_per_frame=max_rois, max_frames=n,
                               keep_mask=1 if keep_mask else 0, max_canvases=self.max_canvases,
                               pitch=self.ring.pitch)
        self.d_cur, self.d_prev = self.ring.tables()
        self.d_ids = ctx.malloc(8 * n)
        self.d_gen = ctx.malloc(8 * n)
        ctx.upload(self.d_ids, np.arange(n, dtype=np.uint64))
        ctx.upload(self.d_gen, np.array(self.t_us, np.int64))
        self.canvas_bytes = canvas[0] * canvas[1] * 3
        self.d_canvases = ctx.malloc(self.canvas_bytes * max(1, self.max_canvases))
        ctx.memset(self.d_canvases, 0xAB, self.canvas_bytes * max(1, self.max_canvases))
        self.first_patch_id = first_patch_id
        self.canvas = canvas
        self.zones, self.radius, self.threshold, self.max_rois = zones, radius, threshold, max_rois

    def run(self):
        self.pipe.run(self.n, self.d_cur, self.d_prev, self.d_ids, self.d_gen, self.first_patch_id,
                      self.d_canvases)
        self.res = self.pipe.results(self.n)
        return self.res

    def canvases(self, count=None):
        count = self.res["total_canvases"] if count is None else count
        return self.ctx.download(self.d_canvases, (count, self.canvas[1], self.canvas[0] * 3),
                                 np.uint8)

    def host_frames(self):
        return [self.ring.download_frame(i) for i in range(self.n + 1)]

    def oracle(self, frames=None, idx=None, lib="port", want_canvases=True):
        frames = frames if frames is not None else self.host_frames()
        idx = list(range(self.n)) if idx is None else idx
        params = oracle_params(self.W, self.H, self.radius, self.threshold, self.zones, self.canvas,
                               self.max_rois, pitch=self.ring.pitch)
        return O.process_frames(params, [frames[i + 1] for i in idx], [frames[i] for i in idx], idx,
                                [self.t_us[i] for i in idx], self.first_patch_id,
                                want_canvases=want_canvases, want_cells=True, lib=lib)

    def close(self):
        self.pipe.close()
        self.ring.close()
        for p in (self.d_ids, self.d_gen, self.d_canvases):
            self.ctx.free(p)


def patch_tuples(plist):
    return [[(p.patch_id, p.source_frame_id, p.rect.x, p.rect.y, p.rect.w, p.rect.h,
              p.generation_time_us, p.slo_us, p.deadline_us, p.size_bytes) for p in fr]
            for fr in plist]


def oracle_patch_tuples(plist):
    return [[(p["patch_id"], p["source_frame_id"], *p["rect"], p["generation_time_us"], p["slo_us"],
              p["deadline_us"], p["size_bytes"]) for p in fr] for fr in plist]
