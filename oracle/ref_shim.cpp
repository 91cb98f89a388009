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
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/partition.hpp"
#include "tangram/rng.hpp"
#include "tangram/scheduler.hpp"
#include "tangram/sim.hpp"
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

// ---- the reference's own simulator, tangram policy (sim.hpp:206-552) ------
// Runs tangram::run() on the given scenes and returns, from its event log,
// every invoke the SloScheduler made plus each patch's admission and arrival
// time from RunMetrics -- the parity target for the device batcher.
typedef struct {
  int32_t width, height, zones_x, zones_y, canvas_w, canvas_h, per_scene_link;
  double vram_per_canvas_gb, gpu_memory_gb, model_size_gb, bandwidth_mbps, bytes_per_pixel;
  int64_t slo_us;
} ref_sim_cfg;

// the event log of the last ref_run_tangram (EventLog JSON lines)
static std::string g_last_log;

int64_t ref_last_log(char* out, int64_t cap) {
  const int64_t n = static_cast<int64_t>(g_last_log.size());
  if (out != nullptr && cap >= n) std::copy(g_last_log.begin(), g_last_log.end(), out);
  return n;
}

int ref_run_tangram(const ref_sim_cfg* c, int n_scenes, const int32_t* frames_per_scene,
                    const int64_t* t_us, const int32_t* roi_counts, const orc_rect* rois,
                    const double* profile, int n_profile, int64_t* arrival_us, uint8_t* admitted,
                    int32_t* n_patches, int64_t patch_cap, int32_t* n_events, int64_t* ev_fire,
                    int32_t* ev_trigger, int32_t* ev_k, int64_t* ev_slack, int32_t* ev_npatch,
                    uint64_t* ev_ids, int64_t ev_cap, int64_t ids_cap, double* eff_mean,
                    double* eff_median) {
  try {
    std::vector<tangram::TraceScene> scenes;
    int64_t fi = 0, ri = 0;
    for (int s = 0; s < n_scenes; ++s) {
      tangram::TraceScene sc;
      sc.scene_id = "cam" + std::to_string(s);
      for (int f = 0; f < frames_per_scene[s]; ++f, ++fi) {
        tangram::TraceFrame tf;
        tf.frame_id = static_cast<uint64_t>(f);
        tf.t_us = t_us[fi];
        tf.width = c->width;
        tf.height = c->height;
        for (int k = 0; k < roi_counts[fi]; ++k, ++ri) tf.rois.push_back(to_rect(rois[ri]));
        sc.frames.push_back(std::move(tf));
      }
      scenes.push_back(std::move(sc));
    }
    tangram::SimConfig cfg;
    cfg.partition = tangram::PartitionConfig{c->zones_x, c->zones_y};
    cfg.canvas.width = c->canvas_w;
    cfg.canvas.height = c->canvas_h;
    cfg.canvas.vram_per_canvas_gb = c->vram_per_canvas_gb;
    cfg.function.gpu_memory_gb = c->gpu_memory_gb;
    cfg.function.model_size_gb = c->model_size_gb;
    cfg.link.bandwidth_mbps = c->bandwidth_mbps;
    cfg.link.bytes_per_pixel = c->bytes_per_pixel;
    cfg.link.per_scene = c->per_scene_link != 0;
    cfg.policy = tangram::Policy::tangram;
    cfg.slo_us = c->slo_us;
    std::vector<tangram::ProfileEntry> entries;
    for (int i = 0; i < n_profile; ++i)
      entries.push_back(tangram::ProfileEntry{static_cast<int>(profile[3 * i]), profile[3 * i + 1],
                                              profile[3 * i + 2]});
    const auto prof = tangram::LatencyProfile::from_entries(c->canvas_w, c->canvas_h, entries);
    std::ostringstream log_text;
    tangram::EventLog log(&log_text, "tangram");
    const tangram::RunMetrics m = tangram::run(scenes, cfg, prof, &log);
    if (static_cast<int64_t>(m.patches.size()) > patch_cap) throw std::length_error("patch cap");
    for (std::size_t i = 0; i < m.patches.size(); ++i) {
      // bit 0: admitted (sim.hpp:262); bit 1: infeasible at arrival (:296-300)
      admitted[i] = static_cast<uint8_t>((m.patches[i].admitted ? 1 : 0) |
                                         (m.patches[i].infeasible_at_arrival ? 2 : 0));
      arrival_us[i] = m.patches[i].admitted ? m.patches[i].arrival_us : -1;
    }
    *n_patches = static_cast<int32_t>(m.patches.size());
    *eff_mean = m.summary.mean_canvas_efficiency;
    *eff_median = m.summary.median_canvas_efficiency;
    g_last_log = log_text.str();
    std::istringstream in(log_text.str());
    std::string line;
    int64_t ne = 0, nid = 0;
    while (std::getline(in, line)) {
      const auto j = nlohmann::json::parse(line);
      if (j.at("event").get<std::string>() != "invoke") continue;
      if (ne >= ev_cap) throw std::length_error("event cap");
      ev_fire[ne] = j.at("t_us").get<int64_t>();
      const std::string trig = j.at("trigger").get<std::string>();
      ev_trigger[ne] = trig == "deadline_timer" ? 0 : trig == "infeasible_arrival" ? 1 : 2;
      ev_k[ne] = j.at("k").get<int32_t>();
      ev_slack[ne] = j.at("slack_us").get<int64_t>();
      const auto ids = j.at("patches");
      ev_npatch[ne] = static_cast<int32_t>(ids.size());
      for (const auto& id : ids) {
        if (nid >= ids_cap) throw std::length_error("ids cap");
        ev_ids[nid++] = id.get<uint64_t>();
      }
      ++ne;
    }
    *n_events = static_cast<int32_t>(ne);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// tangram::save_trace (trace.hpp:79-90) of the given scenes; returns the
// text length (or -1), writing up to cap bytes into out.
int64_t ref_save_trace(int n_scenes, const int32_t* frames_per_scene, const int64_t* t_us,
                       const int32_t* roi_counts, const orc_rect* rois, int width, int height,
                       char* out, int64_t cap) {
  try {
    std::vector<tangram::TraceScene> scenes;
    int64_t fi = 0, ri = 0;
    for (int s = 0; s < n_scenes; ++s) {
      tangram::TraceScene sc;
      sc.scene_id = "cam" + std::to_string(s);
      for (int f = 0; f < frames_per_scene[s]; ++f, ++fi) {
        tangram::TraceFrame tf;
        tf.frame_id = static_cast<uint64_t>(f);
        tf.t_us = t_us[fi];
        tf.width = width;
        tf.height = height;
        for (int k = 0; k < roi_counts[fi]; ++k, ++ri) tf.rois.push_back(to_rect(rois[ri]));
        sc.frames.push_back(std::move(tf));
      }
      scenes.push_back(std::move(sc));
    }
    std::ostringstream os;
    tangram::save_trace(os, scenes);
    const std::string s = os.str();
    if (static_cast<int64_t>(s.size()) <= cap) std::memcpy(out, s.data(), s.size());
    return static_cast<int64_t>(s.size());
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// The reference SloScheduler driven call by call (scheduler_test.cpp style).
struct RefSched {
  tangram::LatencyProfile prof;
  std::unique_ptr<tangram::SloScheduler> s;
  std::vector<tangram::InvokeEvent> events;
};

void* ref_sched_create(int canvas_w, int canvas_h, const double* profile, int n_profile,
                       int max_canvases) {
  try {
    std::vector<tangram::ProfileEntry> entries;
    for (int i = 0; i < n_profile; ++i)
      entries.push_back(tangram::ProfileEntry{static_cast<int>(profile[3 * i]), profile[3 * i + 1],
                                              profile[3 * i + 2]});
    auto* r = new RefSched{tangram::LatencyProfile::from_entries(canvas_w, canvas_h, entries), {}, {}};
    tangram::CanvasSpec spec;
    spec.width = canvas_w;
    spec.height = canvas_h;
    r->s = std::make_unique<tangram::SloScheduler>(spec, &r->prof, max_canvases);
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_sched_destroy(void* h) { delete static_cast<RefSched*>(h); }

int ref_sched_arrival(void* h, const orc_patch* p, int64_t now) {
  auto* r = static_cast<RefSched*>(h);
  try {
    tangram::PatchMeta m;
    m.patch_id = p->patch_id;
    m.source_frame_id = p->source_frame_id;
    m.rect = to_rect(p->rect);
    m.generation_time_us = p->generation_time_us;
    m.slo_us = p->slo_us;
    m.deadline_us = p->deadline_us;
    m.size_bytes = p->size_bytes;
    r->events = r->s->on_patch_arrival(m, now);
    return static_cast<int>(r->events.size());
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int ref_sched_timer(void* h, int64_t now, uint64_t epoch) {
  auto* r = static_cast<RefSched*>(h);
  r->events.clear();
  if (auto ev = r->s->on_timer(now, epoch)) r->events.push_back(std::move(*ev));
  return static_cast<int>(r->events.size());
}

int ref_sched_pending(void* h, int64_t* at, uint64_t* epoch) {
  auto* r = static_cast<RefSched*>(h);
  const auto t = r->s->pending_timer();
  if (!t) return 0;
  *at = t->fire_at_us;
  *epoch = t->epoch;
  return 1;
}

// Event i: header fields, ids (queue order), placements canvas-major in
// placement order, free rects canvas-major in list order.
int ref_sched_event(void* h, int i, int64_t* fire, int32_t* trigger, int32_t* k, int64_t* slack,
                    int32_t* n_ids, uint64_t* ids, orc_placement* placements, int32_t* n_free,
                    orc_free_rect* free_out) {
  auto* r = static_cast<RefSched*>(h);
  if (i < 0 || i >= static_cast<int>(r->events.size())) return -1;
  const auto& e = r->events[static_cast<std::size_t>(i)];
  *fire = e.fire_time_us;
  *trigger = static_cast<int32_t>(e.trigger);
  *k = e.batch_size;
  *slack = e.estimated_slack_us;
  *n_ids = static_cast<int32_t>(e.patch_ids.size());
  for (std::size_t j = 0; j < e.patch_ids.size(); ++j) ids[j] = e.patch_ids[j];
  int np = 0, nf = 0;
  for (std::size_t c = 0; c < e.stitch.canvases.size(); ++c) {
    for (const auto& p : e.stitch.canvases[c].placements)
      placements[np++] = orc_placement{p.patch_id, p.canvas_index, from_rect(p.position), 0};
    for (const auto& fr : e.stitch.canvases[c].free_rects)
      free_out[nf++] = orc_free_rect{from_rect(fr), static_cast<int32_t>(c)};
  }
  *n_free = nf;
  return 0;
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
