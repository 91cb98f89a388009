"""B200-native Tangram frame->canvas path (arXiv 2404.09267).

The hot path runs as hand-written sm_100a CUDA kernels behind the C ABI in
include/tangram_gpu.h; this package is its Python front-end.  Importing it
does not touch the GPU; the first device call loads lib/libtangram_gpu.so
and fails loudly if it is missing (no CPU fallback).
"""
from .api import (CanvasSpec, CanvasState, CapacityError, Context, CudaError, FrameRing,  # noqa: F401
                  FrameSpec, Graph, InvalidArgument, NoDevice, OutOfRange, PartitionConfig,
                  PatchMeta, Pipeline, Placement, Rect, StitchResult, TangramError, area,
                  assign_rois, canvas_efficiency, concat_stitches, contains, default_context,
                  derive_seed, dump_layout, enclosing_rect, extract_canvas, generate_trace,
                  make_zones, overlap_area, partition, stitch_all)

__all__ = [n for n in dir() if not n.startswith("_")]
