"""Data formats and summary metrics around the hot path.

* Trace JSON lines (trace.hpp:73-139): one frame per line,
  ``{"H":..,"W":..,"frame":..,"rois":[[x,y,w,h],..],"scene":"..","t_ms":..}``
  with keys sorted and compact separators (nlohmann::json::dump), scenes
  contiguous, validated like ``validate_scene`` (trace.hpp:52-71).  Lets the
  pipeline export the RoIs it extracts and import PANDA-style traces.
* ``dump_packing_json`` -- the ``tangram dump-packing --json`` layout
  (tools/tangram_main.cpp:225-248).
* ``efficiency_summary`` -- mean / median canvas efficiency as the
  simulator's summary computes them (sim.hpp:540-550).
* ``scene_from_rois`` -- the RoIs the device extracted from pixels as a
  reference trace scene, so ``save_trace`` hands them to the reference's
  own tools (``tangram simulate --trace``).
* ``dump_canvases`` -- raw canvas dumps (HWC uint8) with a SHA-256 manifest
  for cross-checking canvases between runs and builds.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass, field
from typing import Iterable, TextIO

from .api import InvalidArgument, Rect, StitchResult, canvas_efficiency


@dataclass
class TraceFrame:
    frame_id: int = 0
    t_us: int = 0
    width: int = 0
    height: int = 0
    rois: list = field(default_factory=list)


@dataclass
class TraceScene:
    scene_id: str = ""
    frames: list = field(default_factory=list)


def ms_to_us(ms: float) -> int:
    """partition.hpp:34-36 (round half away from zero)."""
    return int(ms * 1000.0 - 0.5) if ms < 0 else int(ms * 1000.0 + 0.5)


def us_to_ms(us: int) -> float:
    return float(us) / 1000.0


def validate_scene(scene: TraceScene) -> None:
    """trace.hpp:52-71, same messages."""
    prev_t = -1
    for f in scene.frames:
        if f.width < 1 or f.height < 1:
            raise InvalidArgument(f"frame dimensions must be positive (scene {scene.scene_id}, "
                                  f"frame {f.frame_id})")
        if f.t_us <= prev_t and prev_t >= 0:
            raise InvalidArgument(f"frame times must be strictly increasing (scene "
                                  f"{scene.scene_id}, frame {f.frame_id})")
        prev_t = f.t_us
        for i, r in enumerate(f.rois):
            r = r if isinstance(r, Rect) else Rect(*r)
            if r.w < 1 or r.h < 1 or r.x < 0 or r.y < 0 or r.right() > f.width or r.top() > f.height:
                raise InvalidArgument(f"roi outside frame (scene {scene.scene_id}, frame "
                                      f"{f.frame_id}, roi {i})")


def _rect_list(r) -> list:
    return [r.x, r.y, r.w, r.h] if isinstance(r, Rect) else list(r)


def save_trace(out: TextIO, scenes: Iterable[TraceScene]) -> None:
    """trace.hpp:79-90."""
    for sc in scenes:
        for f in sc.frames:
            line = {"scene": sc.scene_id, "frame": f.frame_id, "t_ms": us_to_ms(f.t_us),
                    "W": f.width, "H": f.height, "rois": [_rect_list(r) for r in f.rois]}
            out.write(json.dumps(line, sort_keys=True, separators=(",", ":")) + "\n")


def load_trace(inp: TextIO) -> list[TraceScene]:
    """trace.hpp:92-127: blank lines skipped, scenes grouped by contiguous
    "scene" values, every scene validated."""
    scenes: list[TraceScene] = []
    for line_no, line in enumerate(inp, start=1):
        if not line.strip(" \t\r\n"):
            continue
        try:
            j = json.loads(line)
        except json.JSONDecodeError as e:
            raise InvalidArgument(f"bad trace line {line_no}: {e}") from None
        try:
            rois = []
            for r in j["rois"]:
                if not isinstance(r, list) or len(r) != 4:
                    raise InvalidArgument("roi must be [x, y, w, h]")
                rois.append(Rect(*[int(v) for v in r]))
            f = TraceFrame(int(j["frame"]), ms_to_us(float(j["t_ms"])), int(j["W"]), int(j["H"]),
                           rois)
            sid = str(j["scene"])
        except (KeyError, TypeError, ValueError) as e:
            raise InvalidArgument(f"bad trace line {line_no}: {e}") from None
        if not scenes or scenes[-1].scene_id != sid:
            scenes.append(TraceScene(sid, []))
        scenes[-1].frames.append(f)
    for sc in scenes:
        validate_scene(sc)
    return scenes


def dump_packing_json(result: StitchResult) -> str:
    """tools/tangram_main.cpp:225-248 (nlohmann dump(2): sorted keys)."""
    eff = canvas_efficiency(result)
    doc = {"canvas": {"width": result.spec.width, "height": result.spec.height}, "canvases": []}
    for ci, c in enumerate(result.canvases):
        doc["canvases"].append({
            "index": ci, "efficiency": eff[ci],
            "placements": [{"patch": p.patch_id, "x": p.position.x, "y": p.position.y,
                            "w": p.position.w, "h": p.position.h} for p in c.placements],
            "free_rects": [{"x": r.x, "y": r.y, "w": r.w, "h": r.h} for r in c.free_rects]})
    return json.dumps(doc, indent=2, sort_keys=True) + "\n"


def efficiency_summary(stitches: Iterable[StitchResult]) -> dict:
    """Mean and median per-canvas efficiency over every canvas of every
    invocation, as the simulator's summary (sim.hpp:505-550)."""
    effs: list[float] = []
    for s in stitches:
        effs.extend(canvas_efficiency(s))
    if not effs:
        return {"canvases": 0, "mean_canvas_efficiency": 0.0, "median_canvas_efficiency": 0.0}
    total = 0.0
    for e in effs:
        total += e
    effs.sort()
    mid = len(effs) // 2
    median = effs[mid] if len(effs) % 2 == 1 else 0.5 * (effs[mid - 1] + effs[mid])
    return {"canvases": len(effs), "mean_canvas_efficiency": total / len(effs),
            "median_canvas_efficiency": median}


def scene_from_rois(scene_id: str, t_us, rois_per_frame, width: int, height: int,
                    first_frame: int = 0) -> TraceScene:
    """A trace scene (trace.hpp:39-50) of extracted RoIs: frame i has time
    t_us[i] and the (x, y, w, h) boxes rois_per_frame[i]; validated like a
    loaded trace."""
    frames = [TraceFrame(first_frame + i, int(t), int(width), int(height),
                         [r if isinstance(r, Rect) else Rect(*[int(v) for v in r]) for r in rois])
              for i, (t, rois) in enumerate(zip(t_us, rois_per_frame))]
    sc = TraceScene(str(scene_id), frames)
    validate_scene(sc)
    return sc


def canvas_sha256(canvas) -> str:
    """SHA-256 of a canvas's bytes (row-major HWC uint8, rows unpadded)."""
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(canvas, dtype=np.uint8).tobytes()).hexdigest()


def dump_canvases(directory: str, canvases, prefix: str = "canvas") -> dict:
    """Writes canvases[k] (N x 3M uint8 or N x M x 3) as <prefix>_<k>.rgb raw
    files plus manifest.json {"canvases": [{"index", "file", "width",
    "height", "sha256"}]}; returns the manifest."""
    import numpy as np
    os.makedirs(directory, exist_ok=True)
    entries = []
    for k, c in enumerate(canvases):
        c = np.ascontiguousarray(c, dtype=np.uint8)
        h = c.shape[0]
        w = c.shape[1] if c.ndim == 3 else c.shape[1] // 3
        name = f"{prefix}_{k:06d}.rgb"
        with open(os.path.join(directory, name), "wb") as f:
            f.write(c.tobytes())
        entries.append({"index": k, "file": name, "width": int(w), "height": int(h),
                        "sha256": canvas_sha256(c)})
    manifest = {"format": "rgb8 HWC, rows unpadded", "canvases": entries}
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
        f.write("\n")
    return manifest


def verify_canvas_dump(directory: str) -> list[int]:
    """Indices of dumped canvases whose bytes no longer match the manifest."""
    with open(os.path.join(directory, "manifest.json")) as f:
        manifest = json.load(f)
    bad = []
    for e in manifest["canvases"]:
        with open(os.path.join(directory, e["file"]), "rb") as f:
            if hashlib.sha256(f.read()).hexdigest() != e["sha256"]:
                bad.append(e["index"])
    return bad
