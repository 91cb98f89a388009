"""ctypes binding of ``lib/libtangram_gpu.so`` (the C ABI in include/tangram_gpu.h).

The library is built in-tree (``python -m paper_2404_09267_b200.build``).
Loading fails loudly if it is missing: the package has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = os.environ.get("TANGRAM_GPU_LIB") or _build.LIB  # override: build variants

TG_OK = 0
TG_ERR_INVALID_ARGUMENT = 1
TG_ERR_OUT_OF_RANGE = 2
TG_ERR_CAPACITY = 3
TG_ERR_CUDA = 4
TG_ERR_NO_DEVICE = 5
TG_ERR_COMM = 6
TG_OPT_GATHER_GRID = 1
TG_OPT_GATHER_BAND = 2


class tg_rect(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("w", C.c_int32), ("h", C.c_int32)]


class tg_frame_spec(C.Structure):
    _fields_ = [("frame_id", C.c_uint64), ("width", C.c_int32), ("height", C.c_int32),
                ("generation_time_us", C.c_int64), ("slo_us", C.c_int64)]


class tg_partition_config(C.Structure):
    _fields_ = [("zones_x", C.c_int32), ("zones_y", C.c_int32)]


class tg_patch_meta(C.Structure):
    _fields_ = [("patch_id", C.c_uint64), ("source_frame_id", C.c_uint64), ("rect", tg_rect),
                ("generation_time_us", C.c_int64), ("slo_us", C.c_int64),
                ("deadline_us", C.c_int64), ("size_bytes", C.c_int64)]


class tg_canvas_spec(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("vram_per_canvas_gb", C.c_double)]


class tg_placement(C.Structure):
    _fields_ = [("patch_id", C.c_uint64), ("canvas_index", C.c_int32), ("position", tg_rect),
                ("reserved", C.c_int32)]


class tg_free_rect(C.Structure):
    _fields_ = [("rect", tg_rect), ("canvas_index", C.c_int32), ("seq", C.c_int32)]


class tg_pipeline_params(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pitch", C.c_int32),
                ("threshold", C.c_int32), ("dilate_radius", C.c_int32),
                ("partition", tg_partition_config), ("canvas", tg_canvas_spec),
                ("bytes_per_pixel", C.c_double), ("slo_us", C.c_int64),
                ("max_frames", C.c_int32), ("max_rois_per_frame", C.c_int32),
                ("max_canvases", C.c_int64), ("keep_mask", C.c_int32)]


class tg_pipeline_views(C.Structure):
    _fields_ = [("n_rois", C.c_void_p), ("rois", C.c_void_p), ("n_patches", C.c_void_p),
                ("patches", C.c_void_p), ("admitted", C.c_void_p), ("n_placements", C.c_void_p),
                ("placements", C.c_void_p), ("n_canvases", C.c_void_p),
                ("canvas_base", C.c_void_p), ("cells", C.c_void_p), ("mask", C.c_void_p),
                ("zones", C.c_int32), ("cells_x", C.c_int32), ("cells_y", C.c_int32),
                ("mask_words", C.c_int32)]


class tg_pipeline_stats(C.Structure):
    _fields_ = [("mask_fused_launches", C.c_int64), ("mask_split_launches", C.c_int64)]


class tg_workload_config(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("fps", C.c_double), ("frame_width", C.c_int32),
                ("frame_height", C.c_int32), ("roi_proportion_mean", C.c_double),
                ("roi_proportion_jitter", C.c_double), ("burst_probability", C.c_double),
                ("burst_multiplier", C.c_double), ("roi_count_min", C.c_int32),
                ("roi_count_max", C.c_int32), ("roi_aspect_min", C.c_double),
                ("roi_aspect_max", C.c_double), ("roi_max_dim", C.c_int32), ("seed", C.c_uint64)]


class tg_gather_job(C.Structure):
    _fields_ = [("dst", tg_rect), ("src_frame", C.c_int32), ("src_x", C.c_int32),
                ("src_y", C.c_int32)]


class tg_ipc_handle(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 64)]


class tg_comm_id(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 128)]


# tg_host_allgather_fn: (send, bytes, recv, user) -> 0 on success
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class tg_profile_entry(C.Structure):
    _fields_ = [("batch_size", C.c_int32), ("mu_ms", C.c_double), ("sigma_ms", C.c_double)]


class tg_invoke_info(C.Structure):
    _fields_ = [("fire_time_us", C.c_int64), ("batch_size", C.c_int32), ("trigger", C.c_int32),
                ("estimated_slack_us", C.c_int64), ("n_patches", C.c_int32),
                ("n_free", C.c_int32)]


P = C.POINTER
vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
sz = C.c_size_t
st = C.c_int  # tg_status

# name -> (restype, argtypes); every symbol include/tangram_gpu.h declares.
SIGNATURES = {
    "tg_abi_version": (C.c_int, []),
    "tg_last_error": (C.c_char_p, []),
    "tg_device_count": (st, [P(i32)]),
    "tg_ctx_create": (st, [i32, P(vp)]),
    "tg_ctx_destroy": (None, [vp]),
    "tg_ctx_stream": (vp, [vp]),
    "tg_ctx_synchronize": (st, [vp]),
    "tg_device_sm_count": (st, [vp, P(i32)]),
    "tg_ctx_set_option": (st, [vp, i32, i64]),
    "tg_malloc_device": (st, [vp, sz, P(vp)]),
    "tg_free_device": (st, [vp, vp]),
    "tg_malloc_host": (st, [vp, sz, P(vp)]),
    "tg_ipc_export": (st, [vp, vp, P(tg_ipc_handle)]),
    "tg_ipc_import": (st, [vp, P(tg_ipc_handle), P(vp)]),
    "tg_ipc_close": (st, [vp, vp]),
    "tg_free_host": (st, [vp, vp]),
    "tg_memcpy_async": (st, [vp, vp, vp, sz, i32, vp]),
    "tg_memset_async": (st, [vp, vp, i32, sz, vp]),
    "tg_stream_create": (st, [vp, P(vp)]),
    "tg_stream_create_priority": (st, [vp, i32, P(vp)]),
    "tg_stream_destroy": (st, [vp, vp]),
    "tg_stream_synchronize": (st, [vp, vp]),
    "tg_event_create": (st, [vp, P(vp)]),
    "tg_event_destroy": (st, [vp, vp]),
    "tg_event_record": (st, [vp, vp, vp]),
    "tg_event_elapsed_ms": (st, [vp, vp, vp, P(C.c_float)]),
    "tg_stream_wait_event": (st, [vp, vp, vp]),
    "tg_event_synchronize": (st, [vp, vp]),
    "tg_make_zones": (st, [P(tg_frame_spec), tg_partition_config, P(tg_rect), i32]),
    "tg_assign_rois": (st, [vp, P(tg_rect), i32, P(tg_rect), i32, P(i32)]),
    "tg_partition": (st, [vp, P(tg_frame_spec), tg_partition_config, P(tg_rect), i32, C.c_double,
                          u64, P(tg_patch_meta), i32, P(i32)]),
    "tg_stitch_all": (st, [vp, P(tg_patch_meta), i32, tg_canvas_spec, P(tg_placement), P(i32),
                           P(tg_free_rect), i32, P(i32)]),
    "tg_stitch_batch": (st, [vp, i32, i32, vp, vp, tg_canvas_spec, vp, vp, vp, vp, vp]),
    "tg_pipeline_params_default": (st, [i32, i32, P(tg_pipeline_params)]),
    "tg_pipeline_create": (st, [vp, P(tg_pipeline_params), P(vp)]),
    "tg_pipeline_destroy": (None, [vp]),
    "tg_pipeline_run": (st, [vp, i32, vp, vp, vp, vp, u64, vp, vp]),
    "tg_pipeline_stage_mask": (st, [vp, i32, vp, vp, vp]),
    "tg_pipeline_stage_mask_fg": (st, [vp, i32, vp, vp, vp]),
    "tg_pipeline_stage_mask_cells": (st, [vp, i32, vp]),
    "tg_pipeline_stage_plan": (st, [vp, i32, vp, vp, u64, vp]),
    "tg_pipeline_stage_gather": (st, [vp, i32, vp, vp, vp]),
    "tg_pipeline_graph_create": (st, [vp, i32, vp, vp, vp, vp, u64, vp, vp, P(vp)]),
    "tg_graph_launch": (st, [vp, vp]),
    "tg_graph_destroy": (None, [vp]),
    "tg_pipeline_device_views": (st, [vp, P(tg_pipeline_views)]),
    "tg_pipeline_get_stats": (st, [vp, P(tg_pipeline_stats)]),
    "tg_pipeline_download": (st, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, P(i64)]),
    "tg_pipeline_free_rects": (st, [vp, i32, P(tg_free_rect), i32, P(i32)]),
    "tg_stitch_gather": (st, [vp, P(tg_gather_job), i32, P(i32), i32, tg_canvas_spec, vp, i32, vp,
                              vp]),
    "tg_profile_slack_us": (st, [P(tg_profile_entry), i32, i32, P(i64)]),
    "tg_max_canvases_per_batch": (st, [C.c_double, C.c_double, C.c_double, P(i32)]),
    "tg_transmission_schedule": (st, [P(tg_patch_meta), i32, C.c_double, P(i64)]),
    "tg_batcher_create": (st, [tg_canvas_spec, P(tg_profile_entry), i32, i32, P(vp)]),
    "tg_batcher_destroy": (None, [vp]),
    "tg_batcher_set_log": (st, [vp, C.c_char_p]),
    "tg_batcher_take_log": (st, [vp, vp, i64, P(i64)]),
    "tg_batcher_on_patch_arrival": (st, [vp, P(tg_patch_meta), i32, i64, P(i32)]),
    "tg_batcher_on_timer": (st, [vp, i64, u64, P(i32)]),
    "tg_batcher_pending_timer": (st, [vp, P(i32), P(i64), P(u64)]),
    "tg_batcher_status": (st, [vp, P(i32), P(i32), P(i64), P(i64)]),
    "tg_batcher_event": (st, [vp, i32, P(tg_invoke_info), P(u64), P(tg_placement),
                              P(tg_free_rect)]),
    "tg_batcher_current": (st, [vp, P(tg_invoke_info), P(tg_patch_meta), P(tg_placement),
                                P(tg_free_rect)]),
    "tg_batcher_gather": (st, [vp, vp, i32, vp, i32, vp, vp]),
    "tg_batcher_gather_all": (st, [vp, vp, vp, i32, vp, i64, P(i64), vp]),
    "tg_batcher_gather_events": (st, [vp, vp, i32, i32, vp, i32, vp, i64, P(i64), vp]),
    "tg_batcher_replay": (st, [vp, P(tg_patch_meta), P(i32), P(i64), i32, P(i32)]),
    "tg_batcher_replay_links": (st, [vp, i32, vp, vp, vp, C.c_double, i32, vp, P(i32)]),
    "tg_descriptor_block_bytes": (sz, [i64]),
    "tg_pipeline_set_descriptor_output": (st, [vp, vp, i64, vp, i32]),
    "tg_descriptor_blocks_flatten": (st, [vp, i32, i64, vp, i64, P(i64)]),
    "tg_comm_get_unique_id": (st, [P(tg_comm_id)]),
    "tg_comm_create": (st, [vp, P(tg_comm_id), i32, i32, P(vp)]),
    "tg_comm_create_host": (st, [i32, i32, HOST_ALLGATHER_FN, vp, P(vp)]),
    "tg_comm_destroy": (None, [vp]),
    "tg_comm_info": (st, [vp, P(i32), P(i32), P(i32)]),
    "tg_comm_allgather": (st, [vp, vp, sz, vp, vp]),
    "tg_descriptors_allgather": (st, [vp, vp, i64, vp, vp]),
    "tg_descriptors_compact": (st, [vp, vp, vp, i32, vp, i32, i32, vp, i64, P(i64)]),
    "tg_batcher_schedule": (st, [vp, vp, i64, vp, i32, i32, C.c_double, i32, vp, vp, vp, P(i64),
                                 P(i32)]),
    "tg_workload_default": (st, [P(tg_workload_config)]),
    "tg_derive_seed": (u64, [u64, C.c_char_p]),
    "tg_generate_trace": (st, [P(tg_workload_config), P(i64), P(i32), P(tg_rect), i64, P(i64)]),
    "tg_synth_frames": (st, [vp, i32, i32, i32, u64, i32, i32, vp, vp, vp, vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Loads the CUDA library.  Raises if it was never built: there is no
    fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -m paper_2404_09267_b200.build` "
            "(the B200 path has no CPU fallback)")
    dll = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(dll, name)
        fn.restype = res
        fn.argtypes = args
    _lib = dll
    return dll
