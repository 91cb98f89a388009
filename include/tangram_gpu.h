/*
 * tangram_gpu.h -- C ABI of the B200-native Tangram frame->canvas path.
 *
 * The reference (/root/reference/proj/include/tangram) is a header-only C++20
 * library with no FFI of its own; its public surface for this path is the
 * C++ API of partition.hpp and stitch.hpp.  This header is
 * the thin C layer underneath the C++ drop-in (include/tangram/[name].hpp), plus
 * the batched device entry points that carry the data-parallel hot path:
 *
 *   frames -> [K1 mask+cells] -> [K2 RoI boxes, K3 partition, K4 stitch plan,
 *              frame-order prefix] -> [K5 canvas gather]   (all stream-ordered)
 *
 * Conventions
 *   - Plain pointers and sizes only.  "d_" pointers are device memory,
 *     everything else is host memory.
 *   - Every call returns a tg_status.  On failure tg_last_error() returns the
 *     message; messages reuse the reference's exception texts so the C++
 *     drop-in can rethrow the same std::invalid_argument / std::out_of_range.
 *   - Stream-ordered calls take a `void* stream` (a cudaStream_t; NULL = the
 *     context's own stream).  Device-side errors are latched in the context
 *     and reported by the next synchronizing call.
 *   - One context per device; a context is not thread-safe.  Work that uses
 *     a context's or a pipeline's device counters (a pipeline's stages; the
 *     context's explicit-plan gathers tg_stitch_gather / tg_batcher_gather*)
 *     must not run concurrently on two streams: each pipeline, and each
 *     context's gathers, belong to one stream at a time.
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     returns TG_ERR_NO_DEVICE.
 */
#ifndef TANGRAM_GPU_H
#define TANGRAM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 1
#define TG_CELL_SIZE 16   /* patch-grid cell edge in pixels (frozen spec) */
#define TG_CONTINUE_PATCH_IDS (~(uint64_t)0)

typedef enum {
  TG_OK = 0,
  TG_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  TG_ERR_OUT_OF_RANGE = 2,     /* reference: std::out_of_range    */
  TG_ERR_CAPACITY = 3,         /* a fixed device capacity was exceeded */
  TG_ERR_CUDA = 4,             /* CUDA runtime failure */
  TG_ERR_NO_DEVICE = 5,        /* no usable CUDA device: no fallback exists */
  TG_ERR_COMM = 6              /* collective (NCCL / host transport) failure */
} tg_status;

/* ---- POD mirrors of the reference value types --------------------------- */
/* tangram::Rect (geometry.hpp:28-38): bottom-left origin, y up; memory row
 * r of a frame/canvas is reference y = r. */
typedef struct { int32_t x, y, w, h; } tg_rect;

/* tangram::FrameSpec (partition.hpp:40-46) */
typedef struct {
  uint64_t frame_id;
  int32_t width, height;
  int64_t generation_time_us;
  int64_t slo_us;
} tg_frame_spec;

/* tangram::PartitionConfig (partition.hpp:49-52) */
typedef struct { int32_t zones_x, zones_y; } tg_partition_config;

/* tangram::PatchMeta (partition.hpp:56-64), 64 bytes */
typedef struct {
  uint64_t patch_id;
  uint64_t source_frame_id;
  tg_rect rect;
  int64_t generation_time_us;
  int64_t slo_us;
  int64_t deadline_us;
  int64_t size_bytes;
} tg_patch_meta;

/* tangram::CanvasSpec (stitch.hpp:32-40) */
typedef struct {
  int32_t width, height;
  double vram_per_canvas_gb;
} tg_canvas_spec;

/* tangram::Placement (stitch.hpp:42-46), 32 bytes */
typedef struct {
  uint64_t patch_id;
  int32_t canvas_index;
  tg_rect position;
  int32_t reserved;
} tg_placement;

/* One live guillotine free rect (CanvasState::free_rects element,
 * stitch.hpp:48-52).  `seq` is its insertion order: sorting a canvas's
 * rects by seq reproduces the reference's list order. */
typedef struct {
  tg_rect rect;
  int32_t canvas_index;
  int32_t seq;
} tg_free_rect;

typedef struct tg_ctx tg_ctx;
typedef struct tg_pipeline tg_pipeline;
typedef struct tg_graph tg_graph;

/* ---- library / context --------------------------------------------------- */
int tg_abi_version(void);
const char* tg_last_error(void);
tg_status tg_device_count(int32_t* count);
tg_status tg_ctx_create(int32_t device, tg_ctx** out);
void tg_ctx_destroy(tg_ctx* ctx);
void* tg_ctx_stream(tg_ctx* ctx);
tg_status tg_ctx_synchronize(tg_ctx* ctx); /* waits; reports latched device errors */
tg_status tg_device_sm_count(tg_ctx* ctx, int32_t* sms);
/* Context options.  TG_OPT_GATHER_GRID sets the CTAs of the explicit-plan
 * canvas gathers' persistent grid (tg_stitch_gather, tg_batcher_gather*;
 * 0 = SMs x the occupancy limit): below that, the next pass's K1b and
 * planner CTAs co-run with the event gather of configs 3/4 instead of
 * queueing behind it.  TG_OPT_GATHER_BAND sets the canvas rows per
 * (canvas, band) work unit of those gathers (0 = automatic: 64 rows, up to
 * 512 for plans of many canvases). */
typedef enum { TG_OPT_GATHER_GRID = 1, TG_OPT_GATHER_BAND = 2 } tg_option;
tg_status tg_ctx_set_option(tg_ctx* ctx, int32_t option, int64_t value);

/* ---- memory / streams / events (plumbing for callers without a CUDA
 *      runtime of their own) ----------------------------------------------- */
tg_status tg_malloc_device(tg_ctx* ctx, size_t bytes, void** d_ptr);
tg_status tg_free_device(tg_ctx* ctx, void* d_ptr);
tg_status tg_malloc_host(tg_ctx* ctx, size_t bytes, void** h_ptr); /* pinned */
/* Cross-process device memory (global cross-camera mode): a
 * rank exports the base of a tg_malloc_device allocation (its cameras'
 * frame rings); peers import it as a device pointer they can read -- over
 * NVLink from another GPU, or the same memory from another process on this
 * one.  Imported pointers are released with tg_ipc_close. */
typedef struct { uint8_t bytes[64]; } tg_ipc_handle;
tg_status tg_ipc_export(tg_ctx* ctx, void* d_ptr, tg_ipc_handle* out);
tg_status tg_ipc_import(tg_ctx* ctx, const tg_ipc_handle* handle, void** d_ptr);
tg_status tg_ipc_close(tg_ctx* ctx, void* d_ptr);
tg_status tg_free_host(tg_ctx* ctx, void* h_ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device; async on stream */
tg_status tg_memcpy_async(tg_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind,
                          void* stream);
tg_status tg_memset_async(tg_ctx* ctx, void* d_ptr, int32_t value, size_t bytes, void* stream);
tg_status tg_stream_create(tg_ctx* ctx, void** stream);
/* high != 0: the device's greatest stream priority (its CTAs are scheduled
 * ahead of pending CTAs of default-priority streams). */
tg_status tg_stream_create_priority(tg_ctx* ctx, int32_t high, void** stream);
tg_status tg_stream_destroy(tg_ctx* ctx, void* stream);
tg_status tg_stream_synchronize(tg_ctx* ctx, void* stream);
tg_status tg_event_create(tg_ctx* ctx, void** event);
tg_status tg_event_destroy(tg_ctx* ctx, void* event);
tg_status tg_event_record(tg_ctx* ctx, void* event, void* stream);
tg_status tg_event_elapsed_ms(tg_ctx* ctx, void* start, void* stop, float* ms);
tg_status tg_stream_wait_event(tg_ctx* ctx, void* stream, void* event);
tg_status tg_event_synchronize(tg_ctx* ctx, void* event);  /* host waits for the event */

/* ---- drop-in rect-level API (host in, host out, blocking) ----------------
 * Replaces, call for call:
 *   make_zones  partition.hpp:69-88    (host arithmetic)
 *   assign_rois partition.hpp:93-112   (device)
 *   partition   partition.hpp:119-143  (device)
 *   stitch_all  stitch.hpp:108-146     (device, bit-identical placements)   */
tg_status tg_make_zones(const tg_frame_spec* frame, tg_partition_config cfg, tg_rect* zones,
                        int32_t zones_cap);
tg_status tg_assign_rois(tg_ctx* ctx, const tg_rect* rois, int32_t n_rois, const tg_rect* zones,
                         int32_t n_zones, int32_t* zone_of);
tg_status tg_partition(tg_ctx* ctx, const tg_frame_spec* frame, tg_partition_config cfg,
                       const tg_rect* rois, int32_t n_rois, double bytes_per_pixel,
                       uint64_t first_patch_id, tg_patch_meta* patches, int32_t patches_cap,
                       int32_t* n_patches);
/* placements[i] is queue[i]'s placement; free_rects receives every canvas's
 * live free set (canvas-major, each canvas in reference list order). */
tg_status tg_stitch_all(tg_ctx* ctx, const tg_patch_meta* queue, int32_t n,
                        tg_canvas_spec spec, tg_placement* placements, int32_t* n_canvases,
                        tg_free_rect* free_rects, int32_t free_cap, int32_t* n_free);

/* ---- batched device rect-level API (stream-ordered, device buffers) ------
 * Many independent queues stitched at once, one warp per queue.
 * d_queue_offsets[q]..d_queue_offsets[q+1] index d_queue; outputs are
 * indexed the same way; d_n_canvases[q] receives each queue's canvas count
 * (-1 when the queue failed).  total_patches = d_queue_offsets[n_queues].
 * d_free_ws must hold 2*total_patches+n_queues tg_free_rect; queue q's live
 * free rects are d_free_ws[2*offsets[q]+q ..][0 .. d_n_free[q]) (unordered;
 * sort each canvas by seq for the reference order).                        */
tg_status tg_stitch_batch(tg_ctx* ctx, int32_t n_queues, int32_t total_patches,
                          const int32_t* d_queue_offsets, const tg_patch_meta* d_queue,
                          tg_canvas_spec spec, tg_placement* d_placements,
                          int32_t* d_n_canvases, tg_free_rect* d_free_ws, int32_t* d_n_free,
                          void* stream);

/* ---- the hot path: frames -> canvases ------------------------------------ */
typedef struct {
  int32_t width, height;       /* frame size in pixels, width % 16 == 0 */
  int32_t pitch;               /* bytes between rows, % 16 == 0, >= 3*width */
  int32_t threshold;           /* fg if max_c |cur-prev| > threshold (default 25) */
  int32_t dilate_radius;       /* square structuring element radius, 0..8 (default 2) */
  tg_partition_config partition;
  tg_canvas_spec canvas;
  double bytes_per_pixel;      /* PatchMeta::size_bytes model (default 1.5) */
  int64_t slo_us;
  int32_t max_frames;          /* frames per run */
  int32_t max_rois_per_frame;  /* RoI slots per frame (default 1024) */
  int64_t max_canvases;        /* canvases the output buffer holds */
  int32_t keep_mask;           /* 1: also write the dilated bit mask (debug/parity) */
} tg_pipeline_params;

tg_status tg_pipeline_params_default(int32_t width, int32_t height, tg_pipeline_params* out);
tg_status tg_pipeline_create(tg_ctx* ctx, const tg_pipeline_params* params, tg_pipeline** out);
void tg_pipeline_destroy(tg_pipeline* p);

/* Runs every stage for n_frames frames, asynchronously on `stream`.
 * d_cur / d_prev: DEVICE arrays of n_frames device pointers (frame i and its
 * predecessor).  d_frame_ids / d_gen_us: device arrays of n_frames.  Patch
 * ids are numbered from first_patch_id in frame order (sim.hpp:249-251);
 * first_patch_id == TG_CONTINUE_PATCH_IDS continues where the previous run
 * on this pipeline stopped (device-side, so chunked streams need no sync);
 * canvases are numbered in frame order and written to
 * d_canvases + k * canvas.width * canvas.height * 3 (uint8 HWC RGB, every
 * byte written: patch pixels or zero). */
tg_status tg_pipeline_run(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                          const uint8_t* const* d_prev, const uint64_t* d_frame_ids,
                          const int64_t* d_gen_us, uint64_t first_patch_id,
                          uint8_t* d_canvases, void* stream);

/* The same stages one by one (parity tests, profiling).  stage_mask =
 * stage_mask_fg (K1: raw foreground bitmap) + stage_mask_cells (K1b:
 * dilation + cell summaries).  The raw bitmap is sparse (only the 32-byte
 * sectors holding foreground are stored, plus per-row word flags), so a
 * stage_mask_cells reads the bitmap of the pipeline's last stage_mask_fg. */
tg_status tg_pipeline_stage_mask(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                 const uint8_t* const* d_prev, void* stream);
tg_status tg_pipeline_stage_mask_fg(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                    const uint8_t* const* d_prev, void* stream);
tg_status tg_pipeline_stage_mask_cells(tg_pipeline* p, int32_t n_frames, void* stream);
tg_status tg_pipeline_stage_plan(tg_pipeline* p, int32_t n_frames, const uint64_t* d_frame_ids,
                                 const int64_t* d_gen_us, uint64_t first_patch_id, void* stream);
tg_status tg_pipeline_stage_gather(tg_pipeline* p, int32_t n_frames,
                                   const uint8_t* const* d_cur, uint8_t* d_canvases,
                                   void* stream);

/* Captures one tg_pipeline_run into a CUDA graph (same arguments) so a
 * steady-state step is a single graph launch. */
tg_status tg_pipeline_graph_create(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                   const uint8_t* const* d_prev, const uint64_t* d_frame_ids,
                                   const int64_t* d_gen_us, uint64_t first_patch_id,
                                   uint8_t* d_canvases, void* stream, tg_graph** out);
tg_status tg_graph_launch(tg_graph* g, void* stream);
void tg_graph_destroy(tg_graph* g);

/* Device-resident results of the last run (valid until the next run);
 * these feed the batcher / descriptor allgather without a host round trip. */
typedef struct {
  int32_t* n_rois;          /* [max_frames] */
  tg_rect* rois;            /* [max_frames * max_rois_per_frame] */
  int32_t* n_patches;       /* [max_frames] (admitted or not) */
  tg_patch_meta* patches;   /* [max_frames * zones] */
  uint8_t* admitted;        /* [max_frames * zones] */
  int32_t* n_placements;    /* [max_frames] == admitted patches */
  tg_placement* placements; /* [max_frames * zones], canvas_index frame-local */
  int32_t* n_canvases;      /* [max_frames] */
  int64_t* canvas_base;     /* [max_frames + 1] global index of each frame's canvas 0 */
  uint32_t* cells;          /* [max_frames * cells_y * cells_x] packed cell summaries */
  uint32_t* mask;           /* [max_frames * height * ceil(width/32)] if keep_mask */
  int32_t zones, cells_x, cells_y, mask_words;
} tg_pipeline_views;
tg_status tg_pipeline_device_views(tg_pipeline* p, tg_pipeline_views* out);

/* Which mask-stage path ran (host-side launch counts since creation): the
 * fused cooperative K1 + K1b launch, or its two-launch fallback when the
 * device cannot co-schedule one K1 CTA per SM (e.g. a shared GPU).  Graph
 * replays are not counted (the capture is). */
typedef struct {
  int64_t mask_fused_launches;
  int64_t mask_split_launches;
} tg_pipeline_stats;
tg_status tg_pipeline_get_stats(tg_pipeline* p, tg_pipeline_stats* out);

/* Blocking copies of the last run's results to host (waits on `stream`,
 * then reports latched device errors). */
tg_status tg_pipeline_download(tg_pipeline* p, int32_t n_frames, void* stream,
                               int32_t* n_rois, tg_rect* rois, int32_t* n_patches,
                               tg_patch_meta* patches, uint8_t* admitted,
                               int32_t* n_placements, tg_placement* placements,
                               int32_t* n_canvases, int64_t* total_canvases);
/* Free rects of frame f's canvases (canvas-major, reference list order). */
tg_status tg_pipeline_free_rects(tg_pipeline* p, int32_t frame, tg_free_rect* out, int32_t cap,
                                 int32_t* n_out);

/* ---- generic canvas writer ----------------------------------------------
 * K5 on an explicit plan: canvas k is tiled by jobs[canvas_job_offsets[k] ..
 * canvas_job_offsets[k+1]) (placements: src_frame >= 0 indexes d_frames;
 * free rects: src_frame = -1, zero fill).  The jobs of a canvas must tile it
 * exactly (placements + final free rects of a stitch result).  Host arrays
 * are staged and launched on `stream`; returns before the copy completes. */
typedef struct {
  tg_rect dst;        /* canvas rect */
  int32_t src_frame;  /* index into d_frames, -1 = zeros */
  int32_t src_x, src_y;
} tg_gather_job;
tg_status tg_stitch_gather(tg_ctx* ctx, const tg_gather_job* jobs, int32_t n_jobs,
                           const int32_t* canvas_job_offsets, int32_t n_canvases,
                           tg_canvas_spec spec, const uint8_t* const* d_frames, int32_t pitch,
                           uint8_t* d_canvases, void* stream);

/* ---- SLO-aware batcher (scheduler.hpp:79-215, Alg. 2 invoker) ------------
 * Host state machine over patch descriptors, identical in decisions, timer
 * epochs, triggers and stitch results to the reference SloScheduler, with an
 * incremental repack: stitch_all is prefix-consistent, so a tentative arrival
 * is one BSSF placement on the current state (O(free rects)) instead of a
 * full repack of the queue (O(queue x free rects)).  Each event's canvases
 * can be materialized on the device with tg_batcher_gather. */
typedef struct { int32_t batch_size; double mu_ms, sigma_ms; } tg_profile_entry; /* latency.hpp:33-37 */
typedef enum { TG_TRIGGER_DEADLINE_TIMER = 0, TG_TRIGGER_INFEASIBLE_ARRIVAL = 1,
               TG_TRIGGER_MEMORY_CAP = 2 } tg_trigger;                            /* scheduler.hpp:29-33 */
typedef struct {
  int64_t fire_time_us;
  int32_t batch_size;          /* canvases */
  int32_t trigger;             /* tg_trigger */
  int64_t estimated_slack_us;
  int32_t n_patches;           /* patch ids in queue order */
  int32_t n_free;              /* free rects over all canvases */
} tg_invoke_info;
typedef struct tg_batcher tg_batcher;

/* slack_us(k) = ms_to_us(mu_k + 3 sigma_k), interpolated (latency.hpp:78-118) */
tg_status tg_profile_slack_us(const tg_profile_entry* entries, int32_t n, int32_t k,
                              int64_t* slack_us);
/* cost.hpp:107-115 */
tg_status tg_max_canvases_per_batch(double gpu_memory_gb, double model_size_gb,
                                    double vram_per_canvas_gb, int32_t* k);
/* trace.hpp:247-267: per-link FIFO arrival times, patches in generation order */
tg_status tg_transmission_schedule(const tg_patch_meta* patches, int32_t n, double bandwidth_mbps,
                                   int64_t* arrival_us);

tg_status tg_batcher_create(tg_canvas_spec spec, const tg_profile_entry* entries, int32_t n_entries,
                            int32_t max_canvases, tg_batcher** out);
void tg_batcher_destroy(tg_batcher* b);
/* Event log (scheduler.hpp:93-188 through event_log.hpp): with a policy
 * name set, every arrival / repack / invoke / timer_set record the
 * reference SloScheduler writes is appended as its JSON line, byte for byte
 * (NULL turns logging off).  take_log copies the accumulated lines and
 * clears them; out == NULL only reports *len. */
tg_status tg_batcher_set_log(tg_batcher* b, const char* policy);
tg_status tg_batcher_take_log(tg_batcher* b, char* out, int64_t cap, int64_t* len);
/* on_patch_arrival (scheduler.hpp:90-126).  src_frame tags the patch's pixels
 * for tg_batcher_gather.  *n_events (0..2) events become readable through
 * tg_batcher_event(b, 0..n-1) until the next call. */
tg_status tg_batcher_on_patch_arrival(tg_batcher* b, const tg_patch_meta* patch, int32_t src_frame,
                                      int64_t now_us, int32_t* n_events);
/* on_timer (scheduler.hpp:130-135); stale epochs produce no event. */
tg_status tg_batcher_on_timer(tg_batcher* b, int64_t now_us, uint64_t epoch, int32_t* n_events);
tg_status tg_batcher_pending_timer(tg_batcher* b, int32_t* has_timer, int64_t* fire_at_us,
                                   uint64_t* epoch);
tg_status tg_batcher_status(tg_batcher* b, int32_t* queue_len, int32_t* canvases,
                            int64_t* earliest_deadline_us, int64_t* remaining_time_us);
/* Event i of the last call: patch ids (queue order), placements (canvas-major,
 * placement order), free rects (canvas-major, reference list order); arrays
 * may be NULL. */
tg_status tg_batcher_event(tg_batcher* b, int32_t i, tg_invoke_info* info, uint64_t* patch_ids,
                           tg_placement* placements, tg_free_rect* free_rects);
/* The live batch (SloScheduler::queue() / current_stitch(), scheduler.hpp:
 * 137-141): info->n_patches queued patches in queue order, their packing
 * (placements canvas-major, free rects canvas-major in list order);
 * info->batch_size = open canvases; arrays may be NULL (sizes first). */
tg_status tg_batcher_current(tg_batcher* b, tg_invoke_info* info, tg_patch_meta* queue,
                             tg_placement* placements, tg_free_rect* free_rects);
/* Writes event i's canvases: d_frames[src_frame] holds each patch's frame. */
tg_status tg_batcher_gather(tg_ctx* ctx, tg_batcher* b, int32_t i, const uint8_t* const* d_frames,
                            int32_t pitch, uint8_t* d_canvases, void* stream);
/* Writes the canvases of every event of the last call back to back (event
 * order, canvas order) in one launch; *n_canvases receives their count. */
tg_status tg_batcher_gather_all(tg_ctx* ctx, tg_batcher* b, const uint8_t* const* d_frames,
                                int32_t pitch, uint8_t* d_canvases, int64_t canvas_cap,
                                int64_t* n_canvases, void* stream);
/* Same for the events i with i % stride == first (event order): how the
 * ranks of the global cross-camera mode split the invokes between them. */
tg_status tg_batcher_gather_events(tg_ctx* ctx, tg_batcher* b, int32_t first, int32_t stride,
                                   const uint8_t* const* d_frames, int32_t pitch,
                                   uint8_t* d_canvases, int64_t canvas_cap, int64_t* n_canvases,
                                   void* stream);
/* Offline driver of the reference event loop for the tangram policy
 * (sim.hpp:334-342, 425-458): arrivals ordered by (arrival_us, input order),
 * a timer is queued when its epoch is new and loses ties to arrivals.  All
 * events are kept; *n_events is their count (tg_batcher_event reads them). */
tg_status tg_batcher_replay(tg_batcher* b, const tg_patch_meta* patches, const int32_t* src_frames,
                            const int64_t* arrival_us, int32_t n, int32_t* n_events);
/* Multi-camera front end (sim.hpp:274-290): admitted patches camera-major
 * (cam_offsets[n_cams+1]), each camera's in generation order, delivered over
 * one FIFO uplink per camera (per_camera_link = 1) or one shared link sorted
 * by (generation time, patch id); then tg_batcher_replay.  arrival_us_out
 * (optional) receives each patch's arrival time. */
tg_status tg_batcher_replay_links(tg_batcher* b, int32_t n_cams, const int32_t* cam_offsets,
                                  const tg_patch_meta* patches, const int32_t* src_frames,
                                  double bandwidth_mbps, int32_t per_camera_link,
                                  int64_t* arrival_us_out, int32_t* n_events);

/* ---- multi-camera descriptors (configs 3/4, sim.hpp:249-262, 274-290) ----
 * One record per patch of a camera shard: what ranks all-gather and what the
 * batcher consumes.  Never pixels. */
typedef struct {
  tg_patch_meta patch;
  int32_t camera;    /* camera id */
  int32_t frame;     /* frame index within the camera */
  int32_t admitted;  /* w <= M && h <= N (sim.hpp:262) */
  int32_t pad;
} tg_descriptor;     /* 80 B */

/* A descriptor block -- what one rank contributes to the all-gather: this
 * header, then `cap` records.  `count` records are valid. */
typedef struct {
  int64_t count;
  int64_t cap;
  int64_t reserved[8];
} tg_descriptor_header; /* 80 B, one record's size */
size_t tg_descriptor_block_bytes(int64_t cap);

/* Device-side descriptor list.  With an output block attached (device
 * memory of tg_descriptor_block_bytes(cap)), every plan stage of the
 * pipeline writes its run's patches there as dense records: record i is the
 * run's i-th patch in frame, zone order (the reference's scene/frame-ordered
 * patch list, sim.hpp:241-262), patch_id run-local from 0.  The planner's
 * frame-order prefix (decoupled look-back over the frames' patch counts) is
 * the compaction scan, so this costs no extra launch.  Pipeline frame f is
 * frame f % frames_per_camera of camera d_cameras[f / frames_per_camera]
 * (d_cameras: device int32 array; NULL: camera 0, frame f).  A run with
 * more than cap patches latches TG_ERR_CAPACITY.  d_block == NULL detaches. */
tg_status tg_pipeline_set_descriptor_output(tg_pipeline* p, void* d_block, int64_t cap,
                                            const int32_t* d_cameras, int32_t frames_per_camera);
/* Host: concatenates the valid records of n_blocks blocks (each
 * tg_descriptor_block_bytes(cap) bytes, e.g. the all-gathered blocks read
 * back) -- rank-major, which is camera-major under contiguous sharding. */
tg_status tg_descriptor_blocks_flatten(const void* blocks, int32_t n_blocks, int64_t cap,
                                       tg_descriptor* out, int64_t out_cap, int64_t* n_out);

/* ---- the collective: descriptor all-gather --------
 * Replaces the reference's single-process scene loop (sim.hpp:241-272) when
 * cameras are sharded over GPUs.  A device communicator runs NCCL on device
 * buffers (stream-ordered); a host communicator moves host buffers through
 * a caller-supplied all-gather (tests, or any out-of-band transport). */
typedef struct tg_comm tg_comm;
typedef struct { uint8_t bytes[128]; } tg_comm_id; /* ncclUniqueId */
/* Rank 0 creates the id and sends it to every rank out of band. */
tg_status tg_comm_get_unique_id(tg_comm_id* out);
tg_status tg_comm_create(tg_ctx* ctx, const tg_comm_id* id, int32_t rank, int32_t world,
                         tg_comm** out);
/* fn gathers `bytes` from every rank into recv (rank-major); returns 0 on
 * success. */
typedef int32_t (*tg_host_allgather_fn)(const void* send, size_t bytes, void* recv, void* user);
tg_status tg_comm_create_host(int32_t rank, int32_t world, tg_host_allgather_fn fn, void* user,
                              tg_comm** out);
void tg_comm_destroy(tg_comm* comm);
tg_status tg_comm_info(tg_comm* comm, int32_t* rank, int32_t* world, int32_t* on_device);
/* recv (world * bytes) receives every rank's send buffer, rank-major.
 * Device communicator: device buffers, async on `stream`; host
 * communicator: host buffers, blocking. */
tg_status tg_comm_allgather(tg_comm* comm, const void* send, size_t bytes, void* recv,
                            void* stream);
/* Every rank's descriptor block (cap records each) into blocks_out, rank-major. */
tg_status tg_descriptors_allgather(tg_comm* comm, const void* block, int64_t cap,
                                   void* blocks_out, void* stream);

/* Host compaction of per-frame patch slots (patches[F][zones], n_patches[F],
 * admitted[F][zones], as tg_pipeline_views lays them out) into descriptors,
 * frame order then zone order -- the host restatement of the device list
 * above (for callers holding slots on the host).  Pipeline frame f is frame
 * f % frames_per_camera of camera cameras[f / frames_per_camera]
 * (F = n_cams * frames_per_camera).  TG_ERR_CAPACITY if cap is too small. */
tg_status tg_descriptors_compact(const tg_patch_meta* patches, const int32_t* n_patches,
                                 const uint8_t* admitted, int32_t zones, const int32_t* cameras,
                                 int32_t n_cams, int32_t frames_per_camera, tg_descriptor* out,
                                 int64_t cap, int64_t* n_out);
/* Host half of configs 3/4.  `desc` is camera-major (each camera's records
 * in frame, zone order) -- a shard's own list or the all-gathered list of
 * every shard.  Record i gets patch id i (sim.hpp:249-251: ids over every
 * camera of the job); records of cameras outside cameras[0..n_cams) take
 * their id and are skipped; the admitted ones (sim.hpp:262) of the listed
 * cameras, which must appear in `cameras` order, go through
 * tg_batcher_replay_links with pixels at d_frames index
 * slot * (frames_per_camera + 1) + frame + 1 for camera cameras[slot].
 * Optional outputs per admitted patch, in order: its renumbered meta,
 * source frame index and arrival time. */
tg_status tg_batcher_schedule(tg_batcher* b, const tg_descriptor* desc, int64_t n,
                              const int32_t* cameras, int32_t n_cams, int32_t frames_per_camera,
                              double bandwidth_mbps, int32_t per_camera_link,
                              tg_patch_meta* admitted_out, int32_t* src_frames_out,
                              int64_t* arrival_us_out, int64_t* n_admitted, int32_t* n_events);

/* ---- synthetic workload (fixture source; not part of the timed path) -----
 * trace.hpp:145-231 generate_trace, restated (std::mt19937_64 + the
 * reference's hand-rolled distributions).  Writes t_us[n_frames],
 * roi_counts[n_frames] and the RoIs back to back; returns TG_ERR_CAPACITY if
 * roi_cap is too small. */
typedef struct {
  int32_t n_frames;
  double fps;
  int32_t frame_width, frame_height;
  double roi_proportion_mean, roi_proportion_jitter;
  double burst_probability, burst_multiplier;
  int32_t roi_count_min, roi_count_max;
  double roi_aspect_min, roi_aspect_max;
  int32_t roi_max_dim;
  uint64_t seed;
} tg_workload_config;
tg_status tg_workload_default(tg_workload_config* out);
uint64_t tg_derive_seed(uint64_t master, const char* component);
tg_status tg_generate_trace(const tg_workload_config* cfg, int64_t* t_us, int32_t* roi_counts,
                            tg_rect* rois, int64_t roi_cap, int64_t* n_rois_total);
/* Synthesizes frames on the device (frozen pixel spec).
 * Frame i gets time index t0 + i (-1 = background only), its RoIs are
 * d_rects[d_rect_offsets[i] .. d_rect_offsets[i+1]). */
tg_status tg_synth_frames(tg_ctx* ctx, int32_t width, int32_t height, int32_t pitch,
                          uint64_t pixel_seed, int32_t n_frames, int32_t t0,
                          const tg_rect* d_rects, const int32_t* d_rect_offsets,
                          uint8_t* const* d_frames, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TANGRAM_GPU_H */
