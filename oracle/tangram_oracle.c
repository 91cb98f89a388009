/*
 * tangram_oracle.c -- TEST INFRASTRUCTURE ONLY (see tangram_oracle.h).
 *
 * Plain-C restatement of the reference's rect-level algorithms plus the
 * frozen pixel spec.  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/include/tangram/).
 * Compile with -ffp-contract=off so double arithmetic matches the reference
 * build bit-for-bit.
 */
#include "tangram_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static void set_err(const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
}

const char* orc_last_error(void) { return g_err; }
void orc_set_error(const char* msg) { set_err(msg); }

/* ======================================================================== */
/* rng.hpp:27-38  derive_seed: FNV-1a over the name, splitmix64 finalizer.   */
/* ======================================================================== */
uint64_t orc_derive_seed(uint64_t master, const char* component) {
  uint64_t h = 14695981039346656037ull;
  for (const unsigned char* p = (const unsigned char*)component; *p; ++p) {
    h ^= (uint64_t)(*p);
    h *= 1099511628211ull;
  }
  uint64_t z = master + 0x9e3779b97f4a7c15ull + h;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:42-70 wraps std::mt19937_64, whose algorithm is fixed by the C++
 * standard ([rand.predef]: w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29
 * d=0x5555555555555555 s=17 b=0x71d67fffeda60000 t=37 c=0xfff7eee000000000
 * l=43 f=6364136223846793005).  Restated here. */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:47 */
double orc_rng_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:49 */
double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_uniform01(r);
}
/* rng.hpp:52-55 */
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (int64_t)(orc_rng_next(r) % span);
}
/* rng.hpp:58-63 */
double orc_rng_normal(orc_rng* r, double mu, double sigma) {
  double u1 = 1.0 - orc_rng_uniform01(r);
  double u2 = orc_rng_uniform01(r);
  double mag = sqrt(-2.0 * log(u1));
  return mu + sigma * mag * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

/* ======================================================================== */
/* trace.hpp:145-231  synthetic RoI workload                                  */
/* ======================================================================== */
void orc_gen_cfg_default(orc_gen_cfg* c) {
  c->n_frames = 150;
  c->fps = 15.0;
  c->frame_width = 1920;
  c->frame_height = 1080;
  c->roi_proportion_mean = 0.10;
  c->roi_proportion_jitter = 0.5;
  c->burst_probability = 0.05;
  c->burst_multiplier = 3.0;
  c->roi_count_min = 2;
  c->roi_count_max = 12;
  c->roi_aspect_min = 0.5;
  c->roi_aspect_max = 2.0;
  c->roi_max_dim = 480;
  c->seed = 1;
}

/* trace.hpp:162-181 */
static int gen_validate(const orc_gen_cfg* c) {
  if (c->n_frames < 0) return set_err("frame count must be >= 0"), 1;
  if (!(c->fps > 0.0)) return set_err("fps must be positive"), 1;
  if (c->frame_width < 1 || c->frame_height < 1)
    return set_err("frame dimensions must be positive"), 1;
  if (!(c->roi_proportion_mean > 0.0) || c->roi_proportion_mean >= 1.0)
    return set_err("roi proportion must be in (0, 1)"), 1;
  if (c->roi_proportion_jitter < 0.0 || c->roi_proportion_jitter > 1.0)
    return set_err("roi jitter must be in [0, 1]"), 1;
  if (c->burst_probability < 0.0 || c->burst_probability > 1.0)
    return set_err("burst probability must be in [0, 1]"), 1;
  if (c->burst_multiplier < 1.0) return set_err("burst multiplier must be >= 1"), 1;
  if (c->roi_count_min < 0 || c->roi_count_max < c->roi_count_min)
    return set_err("bad roi count range"), 1;
  if (!(c->roi_aspect_min > 0.0) || c->roi_aspect_max < c->roi_aspect_min)
    return set_err("bad roi aspect range"), 1;
  if (c->roi_max_dim < 4) return set_err("roi max dim must be >= 4"), 1;
  if (c->roi_count_max > 0 && (c->frame_width < 4 || c->frame_height < 4))
    return set_err("cannot place requested roi count in frame"), 1;
  return 0;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

int64_t orc_generate_trace(const orc_gen_cfg* cfg, int64_t* t_us, int32_t* roi_counts,
                           orc_rect* rois, int64_t roi_cap) {
  if (gen_validate(cfg)) return -1;
  orc_rng rng;
  orc_rng_seed(&rng, orc_derive_seed(cfg->seed, "trace"));
  int64_t total = 0;
  double* weights = (double*)malloc(sizeof(double) * (size_t)(cfg->roi_count_max + 1));
  for (int i = 0; i < cfg->n_frames; ++i) {
    t_us[i] = llround((double)i * 1e6 / cfg->fps);                       /* :193 */
    const int W = cfg->frame_width, H = cfg->frame_height;
    const int burst = orc_rng_uniform01(&rng) < cfg->burst_probability;  /* :197 */
    const double jitter = orc_rng_uniform(&rng, -1.0, 1.0) * cfg->roi_proportion_jitter;
    double proportion = cfg->roi_proportion_mean * (1.0 + jitter);
    if (burst) proportion *= cfg->burst_multiplier;
    proportion = proportion < 0.0 ? 0.0 : (proportion > 0.6 ? 0.6 : proportion); /* :201 */
    const int n_rois = (int)orc_rng_uniform_int(&rng, cfg->roi_count_min, cfg->roi_count_max);
    roi_counts[i] = 0;
    if (n_rois > 0 && proportion > 0.0) {
      double total_weight = 0.0;
      for (int k = 0; k < n_rois; ++k) {
        weights[k] = orc_rng_uniform(&rng, 0.5, 1.5);
        total_weight += weights[k];
      }
      const double total_area = proportion * (double)W * (double)H;
      const int max_w = cfg->roi_max_dim < W ? cfg->roi_max_dim : W;
      const int max_h = cfg->roi_max_dim < H ? cfg->roi_max_dim : H;
      for (int k = 0; k < n_rois; ++k) {                                 /* :215-225 */
        const double area = total_area * weights[k] / total_weight;
        const double aspect = orc_rng_uniform(&rng, cfg->roi_aspect_min, cfg->roi_aspect_max);
        int w = (int)lround(sqrt(area * aspect));
        int h = (int)lround(sqrt(area / aspect));
        w = clampi(w, 4, max_w);
        h = clampi(h, 4, max_h);
        const int x = (int)orc_rng_uniform_int(&rng, 0, W - w);
        const int y = (int)orc_rng_uniform_int(&rng, 0, H - h);
        if (total >= roi_cap) { free(weights); return -2; }
        rois[total].x = x; rois[total].y = y; rois[total].w = w; rois[total].h = h;
        ++total;
        ++roi_counts[i];
      }
    }
  }
  free(weights);
  return total;
}

/* ======================================================================== */
/* geometry.hpp:40-68, partition.hpp:69-143                                  */
/* ======================================================================== */
static int64_t r_area(orc_rect r) { return (int64_t)r.w * (int64_t)r.h; }

static int64_t r_overlap(orc_rect a, orc_rect b) {                       /* geometry.hpp:44-49 */
  int ar = a.x + a.w, br = b.x + b.w, at = a.y + a.h, bt = b.y + b.h;
  int ow = (ar < br ? ar : br) - (a.x > b.x ? a.x : b.x);
  int oh = (at < bt ? at : bt) - (a.y > b.y ? a.y : b.y);
  if (ow <= 0 || oh <= 0) return 0;
  return (int64_t)ow * (int64_t)oh;
}

int orc_make_zones(int width, int height, int zx, int zy, orc_rect* out) {  /* partition.hpp:69-88 */
  if (zx < 1 || zy < 1 || zx > width || zy > height) {
    set_err("zone grid finer than frame");
    return 1;
  }
  const int zw = width / zx, zh = height / zy;
  int k = 0;
  for (int row = 0; row < zy; ++row) {
    const int y = row * zh;
    const int h = (row == zy - 1) ? height - y : zh;
    for (int col = 0; col < zx; ++col) {
      const int x = col * zw;
      const int w = (col == zx - 1) ? width - x : zw;
      out[k].x = x; out[k].y = y; out[k].w = w; out[k].h = h;
      ++k;
    }
  }
  return 0;
}

int orc_assign_rois(const orc_rect* rois, int n, const orc_rect* zones, int nz,
                    int32_t* zone_of) {                                  /* partition.hpp:93-112 */
  for (int i = 0; i < n; ++i) {
    int64_t best = 0;
    int best_zone = -1;
    for (int z = 0; z < nz; ++z) {
      const int64_t s = r_overlap(rois[i], zones[z]);
      if (s > best) { best = s; best_zone = z; }    /* strict '>' keeps the lowest zone */
    }
    if (best_zone < 0) {
      snprintf(g_err, sizeof(g_err), "roi outside frame (roi index %d)", i);
      return 1;
    }
    zone_of[i] = best_zone;
  }
  return 0;
}

int orc_partition(uint64_t frame_id, int width, int height, int64_t gen_us, int64_t slo_us,
                  int zx, int zy, const orc_rect* rois, int n, double bpp,
                  uint64_t first_patch_id, orc_patch* out) {            /* partition.hpp:119-143 */
  if (zx < 1 || zy < 1 || zx > width || zy > height) {
    set_err("zone grid finer than frame");
    return -1;
  }
  const int nz = zx * zy;
  orc_rect* zones = (orc_rect*)malloc(sizeof(orc_rect) * (size_t)nz);
  int32_t* zone_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  orc_make_zones(width, height, zx, zy, zones);
  if (orc_assign_rois(rois, n, zones, nz, zone_of)) {
    free(zones); free(zone_of);
    return -1;
  }
  int np = 0;
  uint64_t next_id = first_patch_id;
  for (int z = 0; z < nz; ++z) {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0, any = 0;
    for (int i = 0; i < n; ++i) {              /* enclosing_rect over the zone's list */
      if (zone_of[i] != z) continue;
      const orc_rect r = rois[i];
      if (!any) { x0 = r.x; y0 = r.y; x1 = r.x + r.w; y1 = r.y + r.h; any = 1; continue; }
      if (r.x < x0) x0 = r.x;
      if (r.y < y0) y0 = r.y;
      if (r.x + r.w > x1) x1 = r.x + r.w;
      if (r.y + r.h > y1) y1 = r.y + r.h;
    }
    if (!any) continue;
    orc_patch* p = &out[np++];
    memset(p, 0, sizeof(*p));
    p->patch_id = next_id++;
    p->source_frame_id = frame_id;
    p->rect.x = x0; p->rect.y = y0; p->rect.w = x1 - x0; p->rect.h = y1 - y0;
    p->generation_time_us = gen_us;
    p->slo_us = slo_us;
    p->deadline_us = gen_us + slo_us;
    p->size_bytes = (int64_t)ceil((double)r_area(p->rect) * bpp);
  }
  free(zones); free(zone_of);
  return np;
}

/* ======================================================================== */
/* stitch.hpp:66-146  BSSF + guillotine, per-canvas free lists in order      */
/* ======================================================================== */
typedef struct { orc_rect* v; int n, cap; } rect_vec;

static void rv_push(rect_vec* a, orc_rect r) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 8;
    a->v = (orc_rect*)realloc(a->v, sizeof(orc_rect) * (size_t)a->cap);
  }
  a->v[a->n++] = r;
}

static void rv_erase(rect_vec* a, int i) {                    /* order-preserving, :137 */
  memmove(a->v + i, a->v + i + 1, sizeof(orc_rect) * (size_t)(a->n - i - 1));
  --a->n;
}

/* stitch.hpp:86-99: cut along the shorter leftover side, ties cut vertically. */
static void split_free(orc_rect c, int w, int h, rect_vec* out) {
  const int lw = c.w - w, lh = c.h - h;
  orc_rect a, b;
  if (lw <= lh) {
    a.x = c.x + w; a.y = c.y; a.w = lw; a.h = c.h;
    b.x = c.x; b.y = c.y + h; b.w = w; b.h = lh;
  } else {
    a.x = c.x + w; a.y = c.y; a.w = lw; a.h = h;
    b.x = c.x; b.y = c.y + h; b.w = c.w; b.h = lh;
  }
  if (a.w > 0 && a.h > 0) rv_push(out, a);
  if (b.w > 0 && b.h > 0) rv_push(out, b);
}

int orc_stitch_all(const orc_patch* queue, int n, int M, int N, orc_placement* placements,
                   int* n_canvases, orc_free_rect* free_out, int free_cap, int* n_free) {
  rect_vec* canv = (rect_vec*)calloc((size_t)(n > 0 ? n : 1), sizeof(rect_vec));
  int nc = 0, rc = 0;
  for (int i = 0; i < n; ++i) {
    const int w = queue[i].rect.w, h = queue[i].rect.h;
    if (w > M || h > N) {                                       /* :114-118 */
      snprintf(g_err, sizeof(g_err), "patch exceeds canvas (patch %llu, %dx%d)",
               (unsigned long long)queue[i].patch_id, w, h);
      rc = 1;
      goto done;
    }
    int bc = -1, bi = -1, bs = 0;
    for (int ci = 0; ci < nc; ++ci) {                           /* :119-128 */
      for (int fi = 0; fi < canv[ci].n; ++fi) {
        const orc_rect c = canv[ci].v[fi];
        if (c.w < w || c.h < h) continue;
        const int s = (c.w - w) < (c.h - h) ? (c.w - w) : (c.h - h);
        int better;
        if (bc < 0) better = 1;                                 /* candidate_better :72-81 */
        else if (s != bs) better = s < bs;
        else if (ci != bc) better = ci < bc;
        else {
          const orc_rect b = canv[bc].v[bi];
          better = (c.y != b.y) ? c.y < b.y : c.x < b.x;
        }
        if (better) { bc = ci; bi = fi; bs = s; }
      }
    }
    if (bc < 0) {                                               /* :129-135 */
      orc_rect full = {0, 0, M, N};
      rv_push(&canv[nc], full);
      bc = nc++;
      bi = 0;
    }
    const orc_rect chosen = canv[bc].v[bi];
    rv_erase(&canv[bc], bi);
    split_free(chosen, w, h, &canv[bc]);
    placements[i].patch_id = queue[i].patch_id;
    placements[i].canvas_index = bc;
    placements[i].position.x = chosen.x;
    placements[i].position.y = chosen.y;
    placements[i].position.w = w;
    placements[i].position.h = h;
    placements[i].pad_ = 0;
  }
  {
    int k = 0;
    for (int ci = 0; ci < nc; ++ci) {
      for (int fi = 0; fi < canv[ci].n; ++fi) {
        if (free_out) {
          if (k >= free_cap) { set_err("free rect capacity"); rc = 2; goto done; }
          free_out[k].r = canv[ci].v[fi];
          free_out[k].canvas = ci;
        }
        ++k;
      }
    }
    if (n_free) *n_free = k;
    if (n_canvases) *n_canvases = nc;
  }
done:
  for (int ci = 0; ci < (n > 0 ? n : 1); ++ci) free(canv[ci].v);
  free(canv);
  return rc;
}

/* ======================================================================== */
/* Frozen pixel spec.  NOT in the reference.                  */
/* ======================================================================== */
uint32_t orc_hash32(uint32_t x) {        /* "lowbias32" integer mixer */
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

/* Background: 96 + h&63 in [96,159].  Foreground of frame t: 32 + h&15 for
 * even t, 224 - h&15 for odd t.  Temporal noise n in [-3,3] on every byte,
 * result clamped to [0,255].  Every fg/bg and even/odd-fg byte difference is
 * > 40 while bg/bg differences are <= 6, so with T=25 the raw mask is exactly
 * rects(t) ∪ rects(t-1). */
void orc_synth_frame(int W, int H, int pitch, uint64_t pixel_seed, int32_t t,
                     const orc_rect* rects, int n_rects, uint8_t* out) {
  const uint32_t s_bg = (uint32_t)pixel_seed;
  const uint32_t s_fg = orc_hash32(s_bg ^ 0x5bd1e995u);
  const uint32_t tn = orc_hash32((uint32_t)(pixel_seed >> 32) + (uint32_t)t);
  const uint32_t tf = s_fg ^ ((uint32_t)t * 0x9E3779B9u);
  for (int y = 0; y < H; ++y) {
    uint8_t* row = out + (size_t)y * (size_t)pitch;
    for (int x = 0; x < W; ++x) {
      for (int c = 0; c < 3; ++c) {
        const uint32_t idx = (uint32_t)(((uint32_t)y * (uint32_t)W + (uint32_t)x) * 3u + (uint32_t)c);
        const int base = 96 + (int)(orc_hash32(idx ^ s_bg) & 63u);
        const int n = (int)(orc_hash32(idx ^ tn) % 7u) - 3;
        const int v = base + n;
        row[x * 3 + c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
      }
    }
  }
  if (t < 0) return;
  for (int k = 0; k < n_rects; ++k) {
    const orc_rect r = rects[k];
    for (int y = r.y; y < r.y + r.h; ++y) {
      uint8_t* row = out + (size_t)y * (size_t)pitch;
      for (int x = r.x; x < r.x + r.w; ++x) {
        for (int c = 0; c < 3; ++c) {
          const uint32_t idx = (uint32_t)(((uint32_t)y * (uint32_t)W + (uint32_t)x) * 3u + (uint32_t)c);
          const int h = (int)(orc_hash32(idx ^ tf) & 15u);
          const int base = (t & 1) ? 224 - h : 32 + h;
          const int n = (int)(orc_hash32(idx ^ tn) % 7u) - 3;
          const int v = base + n;
          row[x * 3 + c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
      }
    }
  }
}

/* The pixels of `region` of synthetic frame t, exactly as orc_synth_frame
 * would write them, without materializing the frame: a pixel is foreground
 * iff it lies in one of frame t's rects.  Used to compose batched canvases
 * from many cameras' frames (configs 3/4) without holding every frame. */
void orc_synth_rect(int W, int H, uint64_t pixel_seed, int32_t t, const orc_rect* rects,
                    int n_rects, orc_rect region, uint8_t* out, int out_pitch) {
  const uint32_t s_bg = (uint32_t)pixel_seed;
  const uint32_t s_fg = orc_hash32(s_bg ^ 0x5bd1e995u);
  const uint32_t tn = orc_hash32((uint32_t)(pixel_seed >> 32) + (uint32_t)t);
  const uint32_t tf = s_fg ^ ((uint32_t)t * 0x9E3779B9u);
  uint8_t* fg = (uint8_t*)calloc((size_t)(region.w > 0 ? region.w : 1), 1);
  (void)H;
  for (int yy = 0; yy < region.h; ++yy) {
    const int y = region.y + yy;
    memset(fg, 0, (size_t)(region.w > 0 ? region.w : 1));
    if (t >= 0) {
      for (int k = 0; k < n_rects; ++k) {
        const orc_rect r = rects[k];
        if (y < r.y || y >= r.y + r.h) continue;
        const int a = r.x > region.x ? r.x : region.x;
        const int b = (r.x + r.w) < (region.x + region.w) ? (r.x + r.w) : (region.x + region.w);
        for (int x = a; x < b; ++x) fg[x - region.x] = 1;
      }
    }
    uint8_t* row = out + (size_t)yy * (size_t)out_pitch;
    for (int xx = 0; xx < region.w; ++xx) {
      const int x = region.x + xx;
      for (int c = 0; c < 3; ++c) {
        const uint32_t idx = (uint32_t)(((uint32_t)y * (uint32_t)W + (uint32_t)x) * 3u + (uint32_t)c);
        int base;
        if (fg[xx]) {
          const int h = (int)(orc_hash32(idx ^ tf) & 15u);
          base = (t & 1) ? 224 - h : 32 + h;
        } else {
          base = 96 + (int)(orc_hash32(idx ^ s_bg) & 63u);
        }
        const int v = base + (int)(orc_hash32(idx ^ tn) % 7u) - 3;
        row[xx * 3 + c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
      }
    }
  }
  free(fg);
}

/* fg0(x,y) = max_c |cur-prev| > T; fg = square (2r+1)^2 dilation of fg0 with
 * everything outside the frame counted as background. */
void orc_mask(const uint8_t* cur, const uint8_t* prev, int W, int H, int pitch, int T, int r,
              uint32_t* mask) {
  const int nw = (W + 31) / 32;
  uint8_t* fg0 = (uint8_t*)malloc((size_t)W * (size_t)H);
  uint8_t* hd = (uint8_t*)malloc((size_t)W * (size_t)H);
  for (int y = 0; y < H; ++y) {
    const uint8_t* a = cur + (size_t)y * pitch;
    const uint8_t* b = prev + (size_t)y * pitch;
    for (int x = 0; x < W; ++x) {
      int m = 0;
      for (int c = 0; c < 3; ++c) {
        int d = (int)a[3 * x + c] - (int)b[3 * x + c];
        if (d < 0) d = -d;
        if (d > m) m = d;
      }
      fg0[(size_t)y * W + x] = (uint8_t)(m > T);
    }
  }
  for (int y = 0; y < H; ++y) {                          /* horizontal pass */
    const uint8_t* s = fg0 + (size_t)y * W;
    uint8_t* d = hd + (size_t)y * W;
    for (int x = 0; x < W; ++x) {
      uint8_t v = 0;
      const int lo = x - r < 0 ? 0 : x - r, hi = x + r >= W ? W - 1 : x + r;
      for (int k = lo; k <= hi && !v; ++k) v |= s[k];
      d[x] = v;
    }
  }
  memset(mask, 0, sizeof(uint32_t) * (size_t)nw * (size_t)H);
  for (int y = 0; y < H; ++y) {                          /* vertical pass */
    const int lo = y - r < 0 ? 0 : y - r, hi = y + r >= H ? H - 1 : y + r;
    uint32_t* mrow = mask + (size_t)y * nw;
    for (int x = 0; x < W; ++x) {
      uint8_t v = 0;
      for (int k = lo; k <= hi && !v; ++k) v |= hd[(size_t)k * W + x];
      if (v) mrow[x >> 5] |= 1u << (x & 31);
    }
  }
  free(fg0);
  free(hd);
}

void orc_cells(const uint32_t* mask, int W, int H, uint32_t* cells) {
  const int nw = (W + 31) / 32;
  const int cx_n = (W + ORC_CELL - 1) / ORC_CELL, cy_n = (H + ORC_CELL - 1) / ORC_CELL;
  for (int cy = 0; cy < cy_n; ++cy) {
    for (int cx = 0; cx < cx_n; ++cx) {
      int occ = 0, x0 = 99, x1 = -1, y0 = 99, y1 = -1;
      for (int ly = 0; ly < ORC_CELL && cy * ORC_CELL + ly < H; ++ly) {
        const int y = cy * ORC_CELL + ly;
        for (int lx = 0; lx < ORC_CELL && cx * ORC_CELL + lx < W; ++lx) {
          const int x = cx * ORC_CELL + lx;
          if (mask[(size_t)y * nw + (x >> 5)] >> (x & 31) & 1u) {
            ++occ;
            if (lx < x0) x0 = lx;
            if (lx > x1) x1 = lx;
            if (ly < y0) y0 = ly;
            if (ly > y1) y1 = ly;
          }
        }
      }
      cells[(size_t)cy * cx_n + cx] =
          occ ? ((uint32_t)occ | (uint32_t)x0 << 9 | (uint32_t)x1 << 13 | (uint32_t)y0 << 17 |
                 (uint32_t)y1 << 21)
              : 0u;
    }
  }
}

int orc_extract_rois(const uint32_t* cells, int cx_n, int cy_n, orc_rect* rois, int cap) {
  const int nc = cx_n * cy_n;
  uint8_t* seen = (uint8_t*)calloc((size_t)nc, 1);
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * (size_t)nc);
  int nr = 0;
  for (int s = 0; s < nc; ++s) {
    if (!cells[s] || seen[s]) continue;
    int x0 = 1 << 30, y0 = 1 << 30, x1 = -1, y1 = -1, sp = 0;
    stack[sp++] = s;
    seen[s] = 1;
    while (sp) {
      const int i = stack[--sp];
      const int cy = i / cx_n, cx = i % cx_n;
      const uint32_t v = cells[i];
      const int px0 = cx * ORC_CELL + (int)(v >> 9 & 15u), px1 = cx * ORC_CELL + (int)(v >> 13 & 15u);
      const int py0 = cy * ORC_CELL + (int)(v >> 17 & 15u), py1 = cy * ORC_CELL + (int)(v >> 21 & 15u);
      if (px0 < x0) x0 = px0;
      if (px1 > x1) x1 = px1;
      if (py0 < y0) y0 = py0;
      if (py1 > y1) y1 = py1;
      for (int dy = -1; dy <= 1; ++dy) {
        for (int dx = -1; dx <= 1; ++dx) {
          const int ny = cy + dy, nx = cx + dx;
          if (ny < 0 || ny >= cy_n || nx < 0 || nx >= cx_n) continue;
          const int j = ny * cx_n + nx;
          if (cells[j] && !seen[j]) { seen[j] = 1; stack[sp++] = j; }
        }
      }
    }
    if (nr >= cap) { free(seen); free(stack); return -2; }
    rois[nr].x = x0; rois[nr].y = y0; rois[nr].w = x1 - x0 + 1; rois[nr].h = y1 - y0 + 1;
    ++nr;
  }
  free(seen);
  free(stack);
  return nr;
}

void orc_fill_canvas(const uint8_t* frame, int pitch, const orc_patch* patches,
                     const orc_placement* placements, int n, int canvas_index, int M, int N,
                     uint8_t* canvas) {
  memset(canvas, 0, (size_t)M * (size_t)N * 3);
  for (int k = 0; k < n; ++k) {
    if (placements[k].canvas_index != canvas_index) continue;
    const orc_rect src = patches[k].rect, dst = placements[k].position;
    for (int v = 0; v < dst.h; ++v) {
      memcpy(canvas + ((size_t)(dst.y + v) * M + dst.x) * 3,
             frame + (size_t)(src.y + v) * pitch + (size_t)src.x * 3, (size_t)dst.w * 3);
    }
  }
}

/* Canvases of batched invoke events (configs 3/4): canvas k is zero-filled
 * and gets jobs[offsets[k] .. offsets[k+1]) copied in, each job a patch
 * rect of frames[job.frame] placed at (dx, dy).  Canvases are split over
 * `threads` workers. */
typedef struct {
  const uint8_t* const* frames;
  int pitch, M, N, n_canvases, stride, start;
  const orc_fill_job* jobs;
  const int64_t* offsets;
  uint8_t* out;
} fill_jobs_arg;

static void* fill_jobs_worker(void* v) {
  const fill_jobs_arg* a = (const fill_jobs_arg*)v;
  const size_t cb = (size_t)a->M * (size_t)a->N * 3;
  for (int k = a->start; k < a->n_canvases; k += a->stride) {
    uint8_t* canvas = a->out + (size_t)k * cb;
    memset(canvas, 0, cb);
    for (int64_t j = a->offsets[k]; j < a->offsets[k + 1]; ++j) {
      const orc_fill_job J = a->jobs[j];
      const uint8_t* src = a->frames[J.frame];
      for (int v = 0; v < J.h; ++v)
        memcpy(canvas + ((size_t)(J.dy + v) * a->M + J.dx) * 3,
               src + (size_t)(J.sy + v) * a->pitch + (size_t)J.sx * 3, (size_t)J.w * 3);
    }
  }
  return NULL;
}

void orc_fill_jobs(const uint8_t* const* frames, int pitch, const orc_fill_job* jobs,
                   const int64_t* offsets, int n_canvases, int M, int N, uint8_t* out,
                   int threads) {
  const int nt = threads > 0 ? threads : 1;
  fill_jobs_arg* args = (fill_jobs_arg*)calloc((size_t)nt, sizeof(fill_jobs_arg));
  pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
  for (int k = 0; k < nt; ++k) {
    args[k] = (fill_jobs_arg){frames, pitch, M, N, n_canvases, nt, k, jobs, offsets, out};
    if (nt == 1) fill_jobs_worker(&args[k]);
    else pthread_create(&th[k], NULL, fill_jobs_worker, &args[k]);
  }
  if (nt > 1)
    for (int k = 0; k < nt; ++k) pthread_join(th[k], NULL);
  free(th);
  free(args);
}

/* ======================================================================== */
/* Per-frame path: sim.hpp:241-272 (partition + admission :262) and          */
/* sim.hpp:302-332 (one stitch_all per frame, canvases in frame order).      */
/* ======================================================================== */
typedef struct {
  const orc_path_params* p;
  int n_frames, stride, start;
  const uint8_t* const* cur;
  const uint8_t* const* prev;
  const uint64_t* frame_ids;
  const int64_t* gen_us;
  orc_path_out* out;
  orc_partition_fn part;
  orc_stitch_fn stitch;
  int rc;
  char err[256];
} worker_arg;

static void* frame_worker(void* va) {
  worker_arg* a = (worker_arg*)va;
  const orc_path_params* p = a->p;
  const int W = p->width, H = p->height, nz = p->zones_x * p->zones_y;
  const int nw = (W + 31) / 32;
  const int cx_n = (W + ORC_CELL - 1) / ORC_CELL, cy_n = (H + ORC_CELL - 1) / ORC_CELL;
  uint32_t* mask = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nw * (size_t)H);
  uint32_t* cells = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)cx_n * (size_t)cy_n);
  orc_patch* adm = (orc_patch*)malloc(sizeof(orc_patch) * (size_t)nz);
  orc_free_rect* fr = (orc_free_rect*)malloc(sizeof(orc_free_rect) * (size_t)(3 * nz + 4));
  a->rc = 0;
  for (int f = a->start; f < a->n_frames; f += a->stride) {
    orc_path_out* o = a->out;
    orc_mask(a->cur[f], a->prev[f], W, H, p->pitch, p->threshold, p->radius, mask);
    orc_cells(mask, W, H, cells);
    if (o->cells) memcpy(o->cells + (size_t)f * cx_n * cy_n, cells, sizeof(uint32_t) * (size_t)cx_n * cy_n);
    orc_rect* rois = o->rois + (size_t)f * p->max_rois;
    const int nr = orc_extract_rois(cells, cx_n, cy_n, rois, p->max_rois);
    if (nr < 0) { a->rc = 4; snprintf(a->err, sizeof(a->err), "roi capacity exceeded (frame %d)", f); break; }
    o->n_rois[f] = nr;
    orc_patch* pt = o->patches + (size_t)f * nz;
    const int np = a->part(a->frame_ids[f], W, H, a->gen_us[f], p->slo_us, p->zones_x, p->zones_y,
                           rois, nr, p->bytes_per_pixel, 0, pt);
    if (np < 0) { a->rc = 1; snprintf(a->err, sizeof(a->err), "%s", orc_last_error()); break; }
    o->n_patches[f] = np;
    int na = 0;
    for (int j = 0; j < np; ++j) {
      const int ok = pt[j].rect.w <= p->canvas_w && pt[j].rect.h <= p->canvas_h;   /* sim.hpp:262 */
      o->admitted[(size_t)f * nz + j] = (uint8_t)ok;
      if (ok) { adm[na] = pt[j]; adm[na].patch_id = (uint64_t)j; ++na; }          /* local index */
    }
    int nc = 0, nf = 0;
    orc_placement* pl = o->placements + (size_t)f * nz;
    const int src = na ? a->stitch(adm, na, p->canvas_w, p->canvas_h, pl, &nc, fr, 3 * nz + 4, &nf) : 0;
    if (src) { a->rc = src; snprintf(a->err, sizeof(a->err), "%s", orc_last_error()); break; }
    o->n_canvases[f] = nc;
    o->n_placements[f] = na;
  }
  free(mask); free(cells); free(adm); free(fr);
  return NULL;
}

typedef struct {
  const orc_path_params* p;
  int start, stride, n_frames;
  const uint8_t* const* cur;
  orc_path_out* out;
  const int64_t* canvas_base;
} fill_arg;

static void* fill_worker(void* va) {
  fill_arg* a = (fill_arg*)va;
  const orc_path_params* p = a->p;
  const int nz = p->zones_x * p->zones_y;
  orc_patch* adm = (orc_patch*)malloc(sizeof(orc_patch) * (size_t)nz);
  const size_t cbytes = (size_t)p->canvas_w * p->canvas_h * 3;
  for (int f = a->start; f < a->n_frames; f += a->stride) {
    orc_path_out* o = a->out;
    const orc_patch* pt = o->patches + (size_t)f * nz;
    int na = 0;
    for (int j = 0; j < o->n_patches[f]; ++j)
      if (o->admitted[(size_t)f * nz + j]) adm[na++] = pt[j];
    for (int c = 0; c < o->n_canvases[f]; ++c) {
      const int64_t k = a->canvas_base[f] + c;
      if (k >= o->canvas_cap) continue;
      orc_fill_canvas(a->cur[f], p->pitch, adm, o->placements + (size_t)f * nz, na, c,
                      p->canvas_w, p->canvas_h, o->canvases + (size_t)k * cbytes);
    }
  }
  free(adm);
  return NULL;
}

int orc_process_frames_with(const orc_path_params* p, int n_frames, const uint8_t* const* cur,
                            const uint8_t* const* prev, const uint64_t* frame_ids,
                            const int64_t* gen_us, uint64_t first_patch_id, orc_path_out* out,
                            orc_partition_fn part, orc_stitch_fn stitch) {
  if (p->width < 1 || p->height < 1 || p->pitch < 3 * p->width) {
    set_err("bad frame geometry");
    return 1;
  }
  if (!part) part = orc_partition;
  if (!stitch) stitch = orc_stitch_all;
  int nt = p->threads > 0 ? p->threads : 1;
  if (nt > n_frames) nt = n_frames > 0 ? n_frames : 1;
  worker_arg* args = (worker_arg*)calloc((size_t)nt, sizeof(worker_arg));
  pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
  for (int k = 0; k < nt; ++k) {
    args[k] = (worker_arg){p, n_frames, nt, k, cur, prev, frame_ids, gen_us, out, part, stitch, 0, {0}};
    if (nt == 1) frame_worker(&args[k]);
    else pthread_create(&th[k], NULL, frame_worker, &args[k]);
  }
  if (nt > 1)
    for (int k = 0; k < nt; ++k) pthread_join(th[k], NULL);
  int rc = 0;
  for (int k = 0; k < nt; ++k)
    if (args[k].rc && !rc) { rc = args[k].rc; set_err(args[k].err); }
  if (rc) { free(args); free(th); return rc; }

  /* Global numbering: patch ids in frame order (sim.hpp:249-251), canvases in
   * frame order (sim.hpp:309-331). */
  const int nz = p->zones_x * p->zones_y;
  int64_t* canvas_base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_frames + 1));
  uint64_t next_id = first_patch_id;
  int64_t cb = 0;
  for (int f = 0; f < n_frames; ++f) {
    orc_patch* pt = out->patches + (size_t)f * nz;
    orc_placement* pl = out->placements + (size_t)f * nz;
    const uint64_t base = next_id;
    for (int j = 0; j < out->n_patches[f]; ++j) pt[j].patch_id = base + (uint64_t)j;
    for (int k = 0; k < out->n_placements[f]; ++k) pl[k].patch_id = base + pl[k].patch_id;
    next_id += (uint64_t)out->n_patches[f];
    canvas_base[f] = cb;
    cb += out->n_canvases[f];
  }
  out->total_canvases = cb;
  if (out->canvases) {
    fill_arg* fa = (fill_arg*)calloc((size_t)nt, sizeof(fill_arg));
    for (int k = 0; k < nt; ++k) {
      fa[k] = (fill_arg){p, k, nt, n_frames, cur, out, canvas_base};
      if (nt == 1) fill_worker(&fa[k]);
      else pthread_create(&th[k], NULL, fill_worker, &fa[k]);
    }
    if (nt > 1)
      for (int k = 0; k < nt; ++k) pthread_join(th[k], NULL);
    free(fa);
  }
  free(canvas_base);
  free(args);
  free(th);
  return 0;
}

int orc_process_frames(const orc_path_params* p, int n_frames, const uint8_t* const* cur,
                       const uint8_t* const* prev, const uint64_t* frame_ids,
                       const int64_t* gen_us, uint64_t first_patch_id, orc_path_out* out) {
  return orc_process_frames_with(p, n_frames, cur, prev, frame_ids, gen_us, first_patch_id, out,
                                 NULL, NULL);
}
