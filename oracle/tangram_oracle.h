/*
 * tangram_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the Tangram frame->canvas path, used as the parity
 * checker for the B200 kernels.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code.  The
 * product library (paper_2404_09267_b200/lib/libtangram_gpu.so) never links,
 * loads or calls it.
 *
 * Two halves:
 *   1. Rect-level core restated from the reference headers
 *      (/root/reference/proj/include/tangram/{geometry,partition,stitch,
 *      rng,trace}.hpp).  Pinned bit-for-bit against the reference itself,
 *      compiled as-is into oracle/_ref/libtangram_ref.so (see Makefile and
 *      tests/test_oracle_cpu.py) and against the reference's own KATs.
 *   2. Pixel stages (mask, cell occupancy, RoI boxes, canvas fill, synthetic
 *      pixels).  These stages DO NOT EXIST in the reference (SURVEY.md §0.2,
 *      §8 rows A1/A2/A13): their spec is frozen here and in DESIGN.md §3.
 *      Parity for them is "unpinned by the reference"; it is pinned by this
 *      restatement plus its committed golden hashes (tests/golden/).
 */
#ifndef TANGRAM_ORACLE_H
#define TANGRAM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- POD mirrors of the reference value types --------------------------- */
typedef struct { int32_t x, y, w, h; } orc_rect;            /* geometry.hpp:28-38 */

typedef struct {                                             /* partition.hpp:56-64 */
  uint64_t patch_id;
  uint64_t source_frame_id;
  orc_rect rect;
  int64_t generation_time_us;
  int64_t slo_us;
  int64_t deadline_us;
  int64_t size_bytes;
} orc_patch;

typedef struct {                                             /* stitch.hpp:42-46 */
  uint64_t patch_id;
  int32_t canvas_index;
  orc_rect position;
  int32_t pad_;
} orc_placement;

typedef struct { orc_rect r; int32_t canvas; } orc_free_rect;

typedef struct {                                             /* trace.hpp:145-160 */
  int32_t n_frames;
  double fps;
  int32_t frame_width, frame_height;
  double roi_proportion_mean, roi_proportion_jitter;
  double burst_probability, burst_multiplier;
  int32_t roi_count_min, roi_count_max;
  double roi_aspect_min, roi_aspect_max;
  int32_t roi_max_dim;
  uint64_t seed;
} orc_gen_cfg;

/* Status codes shared with the C-ABI: 0 ok, 1 invalid_argument, 2 out_of_range. */
const char* orc_last_error(void);
void orc_set_error(const char* msg);

/* ---- rng.hpp:27-70 ------------------------------------------------------ */
typedef struct { uint64_t mt[312]; int idx; } orc_rng;
uint64_t orc_derive_seed(uint64_t master, const char* component);
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi);
double orc_rng_normal(orc_rng* r, double mu, double sigma);

/* ---- trace.hpp:145-231 --------------------------------------------------- */
void orc_gen_cfg_default(orc_gen_cfg* c);
/* Returns total RoIs written (<= roi_cap), or -1 on a validation error
 * (message via orc_last_error), or -2 when roi_cap is too small. */
int64_t orc_generate_trace(const orc_gen_cfg* cfg, int64_t* t_us, int32_t* roi_counts,
                           orc_rect* rois, int64_t roi_cap);

/* ---- partition.hpp:69-143 ------------------------------------------------ */
int orc_make_zones(int width, int height, int zones_x, int zones_y, orc_rect* out);
/* zone_of[i] = chosen zone for RoI i.  Returns 0 or 1 (invalid_argument). */
int orc_assign_rois(const orc_rect* rois, int n, const orc_rect* zones, int nz, int32_t* zone_of);
/* Returns number of patches (<= zones_x*zones_y) or -1 on error. */
int orc_partition(uint64_t frame_id, int width, int height, int64_t gen_us, int64_t slo_us,
                  int zones_x, int zones_y, const orc_rect* rois, int n, double bpp,
                  uint64_t first_patch_id, orc_patch* out);

/* ---- stitch.hpp:108-146 -------------------------------------------------- */
/* Placements are written in queue order.  free_out receives every canvas's
 * live free list, canvas by canvas, each in the reference's list order.
 * Returns 0, or 1 (invalid_argument: patch exceeds canvas), or 2 (capacity). */
int orc_stitch_all(const orc_patch* queue, int n, int canvas_w, int canvas_h,
                   orc_placement* placements, int* n_canvases, orc_free_rect* free_out,
                   int free_cap, int* n_free);

/* ---- frozen pixel spec (absent from the reference) --------- */
#define ORC_CELL 16
uint32_t orc_hash32(uint32_t x);
/* Frame t of a synthetic camera; t = -1 is the background-only frame. */
void orc_synth_frame(int width, int height, int pitch, uint64_t pixel_seed, int32_t t,
                     const orc_rect* rects, int n_rects, uint8_t* out);
/* Pixels of `region` of frame t (same bytes as orc_synth_frame), rows of
 * out_pitch bytes. */
void orc_synth_rect(int width, int height, uint64_t pixel_seed, int32_t t, const orc_rect* rects,
                    int n_rects, orc_rect region, uint8_t* out, int out_pitch);
/* Dilated foreground mask, one bit per pixel, rows of ceil(W/32) words. */
void orc_mask(const uint8_t* cur, const uint8_t* prev, int width, int height, int pitch,
              int threshold, int radius, uint32_t* mask);
/* Cell summaries: bits 0-8 occupancy, 9-12 x0, 13-16 x1, 17-20 y0, 21-24 y1. */
void orc_cells(const uint32_t* mask, int width, int height, uint32_t* cells);
/* 8-connected components over active cells, ordered by their first cell in
 * raster order; one pixel-tight box per component.  Returns count or -2
 * when cap is exceeded. */
int orc_extract_rois(const uint32_t* cells, int cells_x, int cells_y, orc_rect* rois, int cap);
/* Zero-filled canvas with every placement's source pixels copied in. */
void orc_fill_canvas(const uint8_t* frame, int pitch, const orc_patch* patches,
                     const orc_placement* placements, int n, int canvas_index, int canvas_w,
                     int canvas_h, uint8_t* canvas);

/* Batched event canvases: canvas k = zeros + jobs[offsets[k]..offsets[k+1]). */
typedef struct {
  int32_t frame;      /* index into frames[] */
  int32_t sx, sy;     /* source rect origin in that frame */
  int32_t dx, dy;     /* destination in the canvas */
  int32_t w, h;
} orc_fill_job;
void orc_fill_jobs(const uint8_t* const* frames, int pitch, const orc_fill_job* jobs,
                   const int64_t* offsets, int n_canvases, int canvas_w, int canvas_h, uint8_t* out,
                   int threads);

/* ---- whole per-frame path (sim.hpp:241-332 per-frame items) ------------- */
typedef struct {
  int32_t width, height, pitch;
  int32_t threshold, radius;
  int32_t zones_x, zones_y;
  int32_t canvas_w, canvas_h;
  double bytes_per_pixel;
  int64_t slo_us;
  int32_t max_rois;       /* per frame */
  int32_t threads;        /* worker threads for the batch */
} orc_path_params;

typedef struct {
  /* per frame */
  int32_t* n_rois;        /* [n_frames] */
  orc_rect* rois;         /* [n_frames * max_rois] */
  int32_t* n_patches;     /* [n_frames] all patches (admitted or not) */
  orc_patch* patches;     /* [n_frames * zones] */
  uint8_t* admitted;      /* [n_frames * zones] */
  int32_t* n_canvases;    /* [n_frames] */
  orc_placement* placements; /* [n_frames * zones], one per admitted patch, queue order */
  int32_t* n_placements;  /* [n_frames] */
  uint8_t* canvases;      /* optional: [canvas_cap * canvas_w * canvas_h * 3] */
  int64_t canvas_cap;
  uint32_t* cells;        /* optional: [n_frames * cells_y * cells_x] */
  int64_t total_canvases; /* out */
} orc_path_out;

/* cur[i] / prev[i] point at frame i's pixels and its predecessor.  Patch ids
 * are numbered globally from first_patch_id in frame order (sim.hpp:249-251).
 * Returns 0 or an error code (message via orc_last_error). */
int orc_process_frames(const orc_path_params* p, int n_frames, const uint8_t* const* cur,
                       const uint8_t* const* prev, const uint64_t* frame_ids,
                       const int64_t* gen_us, uint64_t first_patch_id, orc_path_out* out);

/* Rect-level stages are pluggable so oracle/_ref can run the reference's own
 * partition()/stitch_all() inside the same pixel path. */
typedef int (*orc_partition_fn)(uint64_t, int, int, int64_t, int64_t, int, int, const orc_rect*,
                                int, double, uint64_t, orc_patch*);
typedef int (*orc_stitch_fn)(const orc_patch*, int, int, int, orc_placement*, int*,
                             orc_free_rect*, int, int*);
int orc_process_frames_with(const orc_path_params* p, int n_frames, const uint8_t* const* cur,
                            const uint8_t* const* prev, const uint64_t* frame_ids,
                            const int64_t* gen_us, uint64_t first_patch_id, orc_path_out* out,
                            orc_partition_fn part, orc_stitch_fn stitch);

#ifdef __cplusplus
}
#endif
#endif
