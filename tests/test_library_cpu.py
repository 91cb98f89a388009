"""CPU-side checks of the product library (no GPU needed).

* the C-ABI library builds, loads and exports every symbol
  include/tangram_gpu.h declares;
* without a device every compute entry point fails loudly (no fallback);
* host-only pieces (make_zones, generate_trace, derive_seed, value helpers)
  agree with the oracle.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

from oracle import oracle as O
from paper_2404_09267_b200 import _native as N
from paper_2404_09267_b200 import api as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tangram_gpu.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_binding_binds():
    assert header_functions() == sorted(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", N.LIB_PATH]).decode()
    exported = set(re.findall(r" T (tg_[a-z0-9_]+)", out))
    assert set(header_functions()) <= exported


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", N.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_abi_version():
    assert N.lib().tg_abi_version() == 1


def _has_device():
    n = C.c_int32()
    N.lib().tg_device_count(C.byref(n))
    return n.value > 0


@pytest.mark.skipif(_has_device(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(A.NoDevice):
        A.Context(0)
    with pytest.raises(A.NoDevice):
        A.partition(A.FrameSpec(0, 100, 100, 0, 1), A.PartitionConfig(2, 2), [(1, 1, 2, 2)], 1.5)


def test_make_zones_matches_oracle():
    for (w, h, zx, zy) in [(100, 100, 2, 2), (101, 100, 2, 2), (3840, 2160, 4, 4), (1920, 1080, 6, 6),
                           (97, 53, 3, 2)]:
        got = A.make_zones(A.FrameSpec(0, w, h, 0, 1), A.PartitionConfig(zx, zy))
        assert [(r.x, r.y, r.w, r.h) for r in got] == O.make_zones(w, h, zx, zy)
    with pytest.raises(A.InvalidArgument, match="zone grid finer than frame"):
        A.make_zones(A.FrameSpec(0, 3, 3, 0, 1), A.PartitionConfig(4, 4))


def test_generate_trace_matches_oracle(golden):
    for name, t in golden["rect"]["traces"].items():
        t_us, frames = A.generate_trace(**t["cfg"])
        assert t_us == t["t_us"]
        assert [[(r.x, r.y, r.w, r.h) for r in f] for f in frames] == \
            [[tuple(r) for r in f] for f in t["rois"]], name
    with pytest.raises(A.InvalidArgument, match="fps must be positive"):
        A.generate_trace(fps=0.0)


def test_derive_seed_matches_oracle():
    for m in (0, 1, 1000, 2026, 2**63):
        for comp in ("trace", "pixels", "exec", ""):
            assert A.derive_seed(m, comp) == O.derive_seed(m, comp)


def test_value_helpers():
    r = A.StitchResult(A.CanvasSpec(100, 100),
                       [A.CanvasState([A.Placement(0, 0, A.Rect(0, 0, 60, 60))], [], 3600),
                        A.CanvasState([A.Placement(1, 1, A.Rect(0, 0, 50, 50))], [], 2500)])
    r.placement_index = {p.patch_id: p for c in r.canvases for p in c.placements}
    assert A.canvas_efficiency(r) == [0.36, 0.25]
    e = A.extract_canvas(r, 1)
    assert e.canvas_count() == 1 and e.placement_index[1].canvas_index == 0
    with pytest.raises(A.OutOfRange):
        A.extract_canvas(r, 2)
    m = A.concat_stitches([r, e])
    assert m.canvas_count() == 3 and m.placement_index[1].canvas_index == 2
    txt = A.dump_layout(r)
    assert "canvas 1" in txt and "patch 0 at (0,0) 60x60" in txt
    assert A.enclosing_rect([A.Rect(5, 5, 10, 10), A.Rect(30, 10, 30, 20)]) == A.Rect(5, 5, 55, 25)
    with pytest.raises(A.InvalidArgument, match="empty rect set"):
        A.enclosing_rect([])
    assert A.overlap_area(A.Rect(30, 10, 30, 20), A.Rect(0, 0, 50, 50)) == 400
