// kernels.cuh -- launch descriptors shared by the kernels and the C ABI.
#pragma once

#include "common.cuh"

namespace tg {

// ---- K1 (k_mask.cu) --------------------------------------------------------
// Split launches (K1, then K1b): with TG_K1_SPARSE the raw bitmap is sparse --
// K1 stores only the 32-byte sectors (8 words) that hold a foreground bit and
// one flag word per 32 raw words per row (bit i: word i is non-zero), K1b
// loads only flagged words; the unstored words keep stale bits nobody reads.
// d_flags: n_frames * H * raw_flag_words(W) words (null: dense bitmap).
#ifndef TG_K1_SPARSE
#define TG_K1_SPARSE 1
#endif
inline int raw_flag_words(int W) { return TG_K1_SPARSE ? (W + 1023) / 1024 : 0; }
cudaError_t launch_mask_fg(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                           int n_frames, int W, int H, int pitch, int threshold, uint32_t* d_raw,
                           uint32_t* d_flags, int sms, cudaStream_t stream);
// d_zero: H * ceil(W/32) zero words (what K1b reads for columns outside the frame)
cudaError_t launch_dilate_cells(const uint32_t* d_raw, const uint32_t* d_zero,
                                const uint32_t* d_flags, int n_frames,
                                int W, int H, int radius, uint32_t* d_cells, uint32_t* d_active,
                                uint32_t* d_mask, cudaStream_t stream);
// K1 + K1b in one cooperative launch (K1b tasks run beside the stream);
// d_sync: mask_sync_words(H, sms) u32 of scratch; when d_active follows it
// directly (one allocation) a single memset clears both.
size_t mask_sync_words(int H, int sms);
cudaError_t launch_mask_fused(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                              int n_frames, int W, int H, int pitch, int threshold, int radius,
                              uint32_t* d_raw, const uint32_t* d_zero, uint32_t* d_flags,
                              uint32_t* d_cells, uint32_t* d_active, uint32_t* d_mask,
                              uint32_t* d_sync, int sms, cudaStream_t stream);

// ---- K2-K4 per-frame planner + frame-order prefix (k_plan.cu) --------------
struct PlanArgs {
  int n_frames, W, H, X, Y, M, N;
  int cells_x, cells_y, act_words, max_rois, job_cap;
  double bpp;
  int64_t slo_us;
  const uint32_t* cells;
  const uint32_t* active;
  const uint64_t* frame_ids;
  const int64_t* gen_us;
  int32_t* n_rois;
  tg_rect* rois;
  int32_t* n_patches;
  tg_patch_meta* patches;
  uint8_t* admitted;
  int32_t* n_placements;
  tg_placement* placements;
  int32_t* n_canvases;
  Job* jobs;
  uint32_t* canvas_jobs;  // [F][Z] start | count << 16
  // frame-order prefix (global patch ids, canvas numbering), by decoupled
  // look-back between the frames' CTAs
  uint64_t first_id;      // ~0: continue from *id_state
  int64_t max_canvases;
  int nbands;
  int64_t* canvas_base;   // [F + 1]
  uint2* ranges;          // [max_canvases] (first job, job count) in the flat job array
  int32_t* gather_units;  // out: [0] min(total, cap) * nbands; [1], [2] K5 counters := 0
  uint64_t* id_state;     // next patch id after this run
  uint64_t* look;         // [look_cap] look-back words: epoch | flag | patches | canvases
  int look_cap;           // max_frames
  uint32_t* psync;        // [3] frame ticket, finished CTAs, epoch
  // optional dense descriptor list: record i = the run's i-th patch
  tg_descriptor_header* desc_head;  // NULL: no descriptor output
  tg_descriptor* desc;              // desc_head + 1
  int64_t desc_cap;
  const int32_t* desc_cameras;      // camera of frame f: [f / desc_fpc] (NULL: 0)
  int desc_fpc;
  DevError* err;
};

struct PartitionBatchArgs {
  int n_frames, X, Y;
  double bpp;
  const tg_frame_spec* frames;
  const int32_t* roi_offsets;  // [n+1]
  const tg_rect* rois;
  const uint64_t* first_ids;   // [n]
  tg_patch_meta* patches;      // [n * X*Y]
  int32_t* n_patches;
  int32_t* zone_of;            // optional [total rois]
  DevError* err;
};

struct StitchBatchArgs {
  int n_queues, M, N;
  const int32_t* offsets;
  const tg_patch_meta* queue;
  tg_placement* placements;
  int32_t* n_canvases;
  FreeRect* free_ws;   // [2*total + n_queues]
  int32_t* n_free;     // optional [n_queues]
  DevError* err;
};

// stitch_batch_kernel stages queues of up to this many patches (and their
// free sets) in shared memory.
constexpr int kStitchStage = 128;

size_t plan_smem_bytes(int cells_x, int cells_y, int max_rois, int zones);
cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream);
cudaError_t launch_partition_batch(const PartitionBatchArgs& a, cudaStream_t stream);
cudaError_t launch_stitch_batch(const StitchBatchArgs& a, cudaStream_t stream);

// ---- K5 (k_gather.cu) -------------------------------------------------------
// Canvas k is tiled by jobs[ranges[k].x .. ranges[k].x + ranges[k].y),
// sorted by dx; src_frame indexes `frames`.
struct GatherArgs {
  const uint8_t* const* frames;
  int pitch, M, N, nbands, band;  // band: canvas rows per unit (gather_band)
  const Job* jobs;
  const uint2* ranges;
  int32_t* units;         // [0]: (canvas, band) units; [1], [2]: K5's claim and finished-CTA
                          // counters (0 at launch; the last CTA resets them)
  uint8_t* out;
};
// grid_ctas: 0 = the persistent grid of sms x the occupancy limit
cudaError_t launch_gather(const GatherArgs& a, int sms, int grid_ctas, cudaStream_t stream);
int gather_bands(int N, int band);
// Rows per (canvas, band) unit for an explicit plan of n_canvases canvases
// of N rows: the default band, doubled (up to 8x) while the plan keeps at
// least 64 units per SM.
int gather_band(int n_canvases, int N, int sms);
// per-frame pipeline gathers (config 2 K5: 0.667 ms at 64 rows, 0.678 at
// 128, 0.739 at 32)
#ifndef TG_GATHER_DEFAULT_BAND
#define TG_GATHER_DEFAULT_BAND 64
#endif
constexpr int kGatherDefaultBand = TG_GATHER_DEFAULT_BAND;

// ---- synthetic frames (k_synth.cu) -----------------------------------------
struct SynthArgs {
  int W, H, pitch, t0;
  uint64_t seed;
  const tg_rect* rects;
  const int32_t* offsets;
  uint8_t* const* frames;
};
cudaError_t launch_synth(const SynthArgs& a, int n_frames, cudaStream_t stream);

}  // namespace tg
