// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference's own headers (/root/reference/proj/include, read
// in place, never copied) and exposes them through the oracle's POD
// interface, so tests can pin the C restatement (tangram_oracle.c) against
// the real thing and bench.py --impl reference can time the reference's own
// partition()/stitch_all() inside the CPU path.  Built by oracle/Makefile
// into oracle/_ref/libtangram_ref.so; nothing in the product links it.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/partition.hpp"
#include "tangram/rng.hpp"
#include "tangram/stitch.hpp"
#include "tangram/trace.hpp"

extern "C" {
#include "tangram_oracle.h"
}

namespace {
thread_local std::string g_err;

tangram::Rect to_rect(const orc_rect& r) { return tangram::Rect{r.x, r.y, r.w, r.h}; }
orc_rect from_rect(const tangram::Rect& r) { return orc_rect{r.x, r.y, r.w, r.h}; }

int fail(const std::exception& e) {
  g_err = e.what();
  orc_set_error(e.what());
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  return 1;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t master, const char* component) {
  return tangram::derive_seed(master, component);
}

// kind: 0 raw engine words, 1 uniform01, 2 uniform_int(lo,hi), 3 normal(lo=mu,hi=sigma)
void ref_rng_draws(uint64_t seed, int kind, double lo, double hi, int n, double* out_d,
                   uint64_t* out_u) {
  tangram::Rng rng(seed);
  std::mt19937_64 eng(seed);
  for (int i = 0; i < n; ++i) {
    switch (kind) {
      case 0: out_u[i] = eng(); break;
      case 1: out_d[i] = rng.uniform01(); break;
      case 2: out_u[i] = static_cast<uint64_t>(rng.uniform_int(static_cast<int64_t>(lo), static_cast<int64_t>(hi))); break;
      default: out_d[i] = rng.normal(lo, hi); break;
    }
  }
}

int64_t ref_generate_trace(const orc_gen_cfg* c, int64_t* t_us, int32_t* roi_counts,
                           orc_rect* rois, int64_t roi_cap) {
  try {
    tangram::WorkloadGenConfig cfg;
    cfg.n_frames = c->n_frames;
    cfg.fps = c->fps;
    cfg.frame_width = c->frame_width;
    cfg.frame_height = c->frame_height;
    cfg.roi_proportion_mean = c->roi_proportion_mean;
    cfg.roi_proportion_jitter = c->roi_proportion_jitter;
    cfg.burst_probability = c->burst_probability;
    cfg.burst_multiplier = c->burst_multiplier;
    cfg.roi_count_min = c->roi_count_min;
    cfg.roi_count_max = c->roi_count_max;
    cfg.roi_aspect_min = c->roi_aspect_min;
    cfg.roi_aspect_max = c->roi_aspect_max;
    cfg.roi_max_dim = c->roi_max_dim;
    cfg.seed = c->seed;
    const tangram::TraceScene scene = tangram::generate_trace(cfg);
    int64_t k = 0;
    for (std::size_t i = 0; i < scene.frames.size(); ++i) {
      const auto& f = scene.frames[i];
      t_us[i] = f.t_us;
      roi_counts[i] = static_cast<int32_t>(f.rois.size());
      for (const auto& r : f.rois) {
        if (k >= roi_cap) return -2;
        rois[k++] = from_rect(r);
      }
    }
    return k;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int ref_make_zones(int width, int height, int zx, int zy, orc_rect* out) {
  try {
    tangram::FrameSpec fs{0, width, height, 0, 1};
    const auto zones = tangram::make_zones(fs, tangram::PartitionConfig{zx, zy});
    for (std::size_t i = 0; i < zones.size(); ++i) out[i] = from_rect(zones[i]);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_partition(uint64_t frame_id, int width, int height, int64_t gen_us, int64_t slo_us,
                  int zx, int zy, const orc_rect* rois, int n, double bpp,
                  uint64_t first_patch_id, orc_patch* out) {
  try {
    std::vector<tangram::Rect> rs(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) rs[static_cast<std::size_t>(i)] = to_rect(rois[i]);
    tangram::FrameSpec fs{frame_id, width, height, gen_us, slo_us};
    const auto patches = tangram::partition(fs, tangram::PartitionConfig{zx, zy}, rs, bpp,
                                            first_patch_id);
    for (std::size_t i = 0; i < patches.size(); ++i) {
      const auto& p = patches[i];
      out[i] = orc_patch{p.patch_id, p.source_frame_id, from_rect(p.rect), p.generation_time_us,
                         p.slo_us, p.deadline_us, p.size_bytes};
    }
    return static_cast<int>(patches.size());
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int ref_stitch_all(const orc_patch* queue, int n, int M, int N, orc_placement* placements,
                   int* n_canvases, orc_free_rect* free_out, int free_cap, int* n_free) {
  try {
    std::vector<tangram::PatchMeta> q(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      auto& p = q[static_cast<std::size_t>(i)];
      p.patch_id = queue[i].patch_id;
      p.source_frame_id = queue[i].source_frame_id;
      p.rect = to_rect(queue[i].rect);
      p.generation_time_us = queue[i].generation_time_us;
      p.slo_us = queue[i].slo_us;
      p.deadline_us = queue[i].deadline_us;
      p.size_bytes = queue[i].size_bytes;
    }
    tangram::CanvasSpec spec;
    spec.width = M;
    spec.height = N;
    const tangram::StitchResult r = tangram::stitch_all(q, spec);
    // Placements in queue order (the map is keyed by id; ids may repeat in
    // hand-made queues, so walk the canvases in placement order instead).
    std::vector<std::size_t> cursor(r.canvases.size(), 0);
    int k = 0;
    {
      // Reconstruct queue order: patch i landed on the canvas whose next
      // unconsumed placement has patch_id == queue[i].patch_id.
      for (int i = 0; i < n; ++i) {
        bool found = false;
        for (std::size_t c = 0; c < r.canvases.size() && !found; ++c) {
          const auto& pl = r.canvases[c].placements;
          if (cursor[c] < pl.size() && pl[cursor[c]].patch_id == queue[i].patch_id) {
            const auto& p = pl[cursor[c]++];
            placements[i] = orc_placement{p.patch_id, p.canvas_index, from_rect(p.position), 0};
            found = true;
          }
        }
        if (!found) throw std::logic_error("placement order reconstruction failed");
      }
    }
    for (std::size_t c = 0; c < r.canvases.size(); ++c) {
      for (const auto& fr : r.canvases[c].free_rects) {
        if (free_out) {
          if (k >= free_cap) throw std::length_error("free rect capacity");
          free_out[k] = orc_free_rect{from_rect(fr), static_cast<int32_t>(c)};
        }
        ++k;
      }
    }
    if (n_free) *n_free = k;
    if (n_canvases) *n_canvases = r.canvas_count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference CPU implementation of the whole per-frame path: the pixel
// stages are the frozen restatement (they are absent from the reference),
// partition() and stitch_all() are the reference's own code.
int ref_process_frames(const orc_path_params* p, int n_frames, const uint8_t* const* cur,
                       const uint8_t* const* prev, const uint64_t* frame_ids,
                       const int64_t* gen_us, uint64_t first_patch_id, orc_path_out* out) {
  const int rc = orc_process_frames_with(p, n_frames, cur, prev, frame_ids, gen_us,
                                         first_patch_id, out, ref_partition, ref_stitch_all);
  if (rc) g_err = orc_last_error();
  return rc;
}

}  // extern "C"
