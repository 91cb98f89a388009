"""Trace JSONL, dump-packing JSON and efficiency summary."""
import io
import json

import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from paper_2404_09267_b200 import formats as Fm
from tests.test_batcher_cpu import SIM_PROFILE, our_run, scenes_for

need_ref = pytest.mark.skipif(not O.have_ref(), reason="reference build (oracle/_ref) absent")


def to_scenes(raw, W, H):
    return [Fm.TraceScene(f"cam{s}", [Fm.TraceFrame(i, t, W, H, [A.Rect(*r) for r in rois])
                                      for i, (t, rois) in enumerate(zip(t_us, frames))])
            for s, (t_us, frames) in enumerate(raw)]


@need_ref
def test_save_trace_byte_identical_to_reference():
    for W, H, kw in [(1920, 1080, {}), (3840, 2160, dict(roi_max_dim=1024))]:
        raw = scenes_for(3, 20, W, H, **kw)
        buf = io.StringIO()
        Fm.save_trace(buf, to_scenes(raw, W, H))
        assert buf.getvalue() == O.save_trace_ref(raw, W, H)


def test_trace_round_trip_and_validation():
    raw = scenes_for(2, 10, 640, 480, roi_max_dim=200)
    scenes = to_scenes(raw, 640, 480)
    buf = io.StringIO()
    Fm.save_trace(buf, scenes)
    back = Fm.load_trace(io.StringIO(buf.getvalue()))
    assert [(s.scene_id, [(f.frame_id, f.t_us, f.width, f.height, f.rois) for f in s.frames])
            for s in back] == \
        [(s.scene_id, [(f.frame_id, f.t_us, f.width, f.height, f.rois) for f in s.frames])
         for s in scenes]
    with pytest.raises(A.InvalidArgument, match="bad trace line 1"):
        Fm.load_trace(io.StringIO("{not json\n"))
    bad = '{"H":10,"W":10,"frame":0,"rois":[[8,8,5,5]],"scene":"s","t_ms":0.0}\n'
    with pytest.raises(A.InvalidArgument, match=r"roi outside frame \(scene s, frame 0, roi 0\)"):
        Fm.load_trace(io.StringIO(bad))
    two = ('{"H":10,"W":10,"frame":0,"rois":[],"scene":"s","t_ms":5.0}\n'
           '{"H":10,"W":10,"frame":1,"rois":[],"scene":"s","t_ms":5.0}\n')
    with pytest.raises(A.InvalidArgument, match="frame times must be strictly increasing"):
        Fm.load_trace(io.StringIO(two))


def test_dump_packing_json_layout():
    r = A.StitchResult(A.CanvasSpec(100, 100),
                       [A.CanvasState([A.Placement(0, 0, A.Rect(0, 0, 60, 60))],
                                      [A.Rect(60, 0, 40, 100), A.Rect(0, 60, 60, 40)], 3600)])
    doc = json.loads(Fm.dump_packing_json(r))
    assert doc["canvas"] == {"height": 100, "width": 100}
    c = doc["canvases"][0]
    assert c["index"] == 0 and c["efficiency"] == 0.36
    assert c["placements"] == [{"h": 60, "patch": 0, "w": 60, "x": 0, "y": 0}]
    assert c["free_rects"][0] == {"h": 100, "w": 40, "x": 60, "y": 0}


@need_ref
def test_efficiency_summary_matches_reference_simulator():
    W, H = 3840, 2160
    raw = scenes_for(5, 24, W, H, roi_max_dim=480)
    ref = O.run_tangram(raw, W, H, SIM_PROFILE, bandwidth_mbps=80.0)
    _, _, events = our_run(raw, W, H, SIM_PROFILE, 80.0)
    s = Fm.efficiency_summary(e.stitch for e in events)
    assert s["mean_canvas_efficiency"] == ref["mean_canvas_efficiency"]
    assert s["median_canvas_efficiency"] == ref["median_canvas_efficiency"]


@need_ref
def test_extracted_rois_export_as_reference_trace():
    """scene_from_rois + save_trace: byte-identical to the reference's own
    save_trace on the same RoIs, and loadable back."""
    W, H = 1920, 1080
    raw = scenes_for(2, 12, W, H)
    scenes = [Fm.scene_from_rois(f"cam{s}", t_us, frames, W, H) for s, (t_us, frames) in
              enumerate(raw)]
    buf = io.StringIO()
    Fm.save_trace(buf, scenes)
    assert buf.getvalue() == O.save_trace_ref(raw, W, H)
    back = Fm.load_trace(io.StringIO(buf.getvalue()))
    assert [[f.rois for f in s.frames] for s in back] == [[f.rois for f in s.frames] for s in scenes]
    with pytest.raises(A.InvalidArgument, match="roi outside frame"):
        Fm.scene_from_rois("x", [0], [[(1900, 0, 40, 10)]], W, H)


def test_canvas_dump_manifest(tmp_path):
    import hashlib

    import numpy as np
    rng = np.random.default_rng(3)
    canv = rng.integers(0, 256, (3, 64, 96 * 3), dtype=np.uint8)
    man = Fm.dump_canvases(str(tmp_path), canv)
    assert [e["sha256"] for e in man["canvases"]] == \
        [hashlib.sha256(c.tobytes()).hexdigest() for c in canv]
    assert man["canvases"][0]["width"] == 96 and man["canvases"][0]["height"] == 64
    assert Fm.verify_canvas_dump(str(tmp_path)) == []
    with open(tmp_path / man["canvases"][1]["file"], "r+b") as f:
        f.write(b"\x00\x01")
    assert Fm.verify_canvas_dump(str(tmp_path)) == [1]
