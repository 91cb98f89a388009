// batcher.cu -- SLO-aware batching invoker (Alg. 2, scheduler.hpp:79-215),
// its arrival model (trace.hpp:247-267), latency estimator (latency.hpp:
// 78-118), memory cap (cost.hpp:107-115), and the generic canvas writer the
// invoke events feed (tg_stitch_gather -> K5 on the device).
//
// The scheduler is host code over descriptors only -- pixels never leave the
// device.  Its decisions are identical to the reference's, but a tentative
// arrival costs one BSSF placement on the live packing instead of a full
// stitch_all() of the queue: stitch_all is prefix-consistent (SURVEY
// Appendix P4; SPEC.md:197 allows incremental placement when identical), so
// stitch_all(Q + [p]) == place(p, stitch_all(Q)).  Free lists keep the
// reference's order (erase in place, append split pieces), so every event's
// StitchResult matches the reference field for field.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <optional>
#include <string>
#include <tuple>
#include <vector>

#include "kernels.cuh"
#include "tangram_gpu.h"

using namespace tg;

// Shared with api.cu (the context and the error slot live there).
extern "C" void tg_internal_set_error(const char* msg);
extern "C" tg_status tg_internal_run_gather(tg_ctx* ctx, const void* jobs, int32_t n_jobs,
                                            const void* ranges, int32_t n_canvases,
                                            tg_canvas_spec spec, const uint8_t* const* d_frames,
                                            int32_t pitch, uint8_t* d_out, void* stream);

namespace {

tg_status bfail(tg_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  tg_internal_set_error(buf);
  return s;
}

int64_t ms_to_us(double ms) {  // partition.hpp:34-36
  return static_cast<int64_t>(ms < 0 ? ms * 1000.0 - 0.5 : ms * 1000.0 + 0.5);
}

// ---- latency.hpp:44-118 -----------------------------------------------------
struct Profile {
  std::vector<tg_profile_entry> e;  // sorted by batch size

  static tg_status make(const tg_profile_entry* in, int n, Profile* out) {
    if (n <= 0) return bfail(TG_ERR_INVALID_ARGUMENT, "latency profile has no entries");
    std::vector<tg_profile_entry> es(in, in + n);
    std::sort(es.begin(), es.end(), [](const tg_profile_entry& a, const tg_profile_entry& b) {
      return a.batch_size < b.batch_size;
    });
    for (size_t i = 0; i < es.size(); ++i) {
      if (es[i].batch_size < 1) return bfail(TG_ERR_INVALID_ARGUMENT, "profile entry with batch size < 1");
      if (es[i].mu_ms <= 0) return bfail(TG_ERR_INVALID_ARGUMENT, "profile entry with non-positive mu");
      if (es[i].sigma_ms < 0) return bfail(TG_ERR_INVALID_ARGUMENT, "profile entry with negative sigma");
      if (i > 0 && es[i - 1].batch_size == es[i].batch_size)
        return bfail(TG_ERR_INVALID_ARGUMENT, "duplicate profile entry for batch size %d",
                     es[i].batch_size);
    }
    out->e = std::move(es);
    return TG_OK;
  }

  // mu + 3 sigma, linear interpolation / extrapolation on slack values,
  // clamped at zero.
  double slack_ms(int k) const {
    auto val = [](const tg_profile_entry& x) { return x.mu_ms + 3.0 * x.sigma_ms; };
    if (e.size() == 1) return val(e[0]);
    auto it = std::lower_bound(e.begin(), e.end(), k, [](const tg_profile_entry& x, int key) {
      return x.batch_size < key;
    });
    const tg_profile_entry *lo, *hi;
    if (it == e.begin()) {
      lo = &e[0];
      hi = &e[1];
    } else if (it == e.end()) {
      lo = &e[e.size() - 2];
      hi = &e[e.size() - 1];
    } else if (it->batch_size == k) {
      return val(*it);
    } else {
      hi = &*it;
      lo = hi - 1;
    }
    const double t = static_cast<double>(k - lo->batch_size) /
                     static_cast<double>(hi->batch_size - lo->batch_size);
    return std::max(0.0, val(*lo) + t * (val(*hi) - val(*lo)));
  }

  int64_t slack_us(int k) const { return ms_to_us(slack_ms(k)); }
};

// ---- incremental guillotine packing (stitch.hpp:66-146) ---------------------
struct Placed {
  tg_placement pl;
  int queue_index;
};

struct CanvasSt {
  std::vector<tg_rect> free;  // reference list order
  std::vector<Placed> placed;
  int64_t used = 0;
};

struct Packing {
  std::vector<CanvasSt> canvases;
  // per canvas (max free-rect width) << 16 | (max free-rect height), kept
  // contiguous so choose() skips canvases nothing fits in without touching them
  std::vector<uint32_t> bound;

  void refresh_bound(int ci) {
    int mw = 0, mh = 0;
    for (const tg_rect& r : canvases[ci].free) {
      mw = std::max(mw, r.w);
      mh = std::max(mh, r.h);
    }
    bound[ci] = static_cast<uint32_t>(mw) << 16 | static_cast<uint32_t>(mh);
  }
};

struct Choice {
  int canvas, fi;  // fi < 0: a new canvas
  tg_rect chosen;
};

// BSSF over every free rect of every open canvas; ties by canvas, y, x
// (candidate_better, stitch.hpp:72-81).
Choice choose(const Packing& st, int w, int h, int M, int N) {
  // One 128-bit key per candidate, (score, canvas, y, x) from the top 32
  // bits down, so the minimum key is the candidate_better winner for any
  // canvas count; infeasible rects get all ones.  The scan is a branch-free
  // min; free rects of a canvas are disjoint, so (canvas, y, x) names the
  // winner, found again in its canvas's list afterwards.
  using u128 = unsigned __int128;
  const u128 none = ~static_cast<u128>(0);
  u128 best = none;
  for (int ci = 0; ci < static_cast<int>(st.canvases.size()); ++ci) {
    const uint32_t bd = st.bound[ci];
    if (static_cast<int>(bd >> 16) < w || static_cast<int>(bd & 0xffff) < h) continue;
    const tg_rect* fr = st.canvases[ci].free.data();
    const int nf = static_cast<int>(st.canvases[ci].free.size());
    const u128 cbits = static_cast<u128>(static_cast<uint32_t>(ci)) << 64;
    for (int fi = 0; fi < nf; ++fi) {
      const tg_rect c = fr[fi];
      const int dw = c.w - w, dh = c.h - h;
      // all ones when the patch does not fit (dw or dh negative): no branch
      const u128 bad = static_cast<u128>(static_cast<__int128>(static_cast<int64_t>(dw | dh) >> 63));
      const u128 s = static_cast<u128>(static_cast<uint32_t>(dw < dh ? dw : dh));
      const u128 key = (s << 96 | cbits | static_cast<u128>(static_cast<uint32_t>(c.y)) << 32 |
                        static_cast<u128>(static_cast<uint32_t>(c.x))) | bad;
      best = key < best ? key : best;
    }
  }
  if (best == none) return Choice{static_cast<int>(st.canvases.size()), -1, tg_rect{0, 0, M, N}};
  const int ci = static_cast<int>(static_cast<uint32_t>(best >> 64));
  const int by = static_cast<int>(static_cast<uint32_t>(best >> 32));
  const int bx = static_cast<int>(static_cast<uint32_t>(best));
  const auto& fr = st.canvases[ci].free;
  int fi = 0;
  while (fr[fi].x != bx || fr[fi].y != by) ++fi;
  return Choice{ci, fi, fr[fi]};
}

void commit(Packing& st, const Choice& ch, const tg_patch_meta& p, int queue_index, int M, int N) {
  if (ch.fi < 0) {
    st.canvases.emplace_back();
    st.canvases.back().free.push_back(tg_rect{0, 0, M, N});
    st.bound.push_back(0);
  }
  CanvasSt& cv = st.canvases[ch.canvas];
  const int fi = ch.fi < 0 ? 0 : ch.fi;
  const tg_rect c = cv.free[fi];
  cv.free.erase(cv.free.begin() + fi);
  const int w = p.rect.w, h = p.rect.h, lw = c.w - w, lh = c.h - h;
  tg_rect a, b;  // split_free_rect, stitch.hpp:86-99
  if (lw <= lh) {
    a = tg_rect{c.x + w, c.y, lw, c.h};
    b = tg_rect{c.x, c.y + h, w, lh};
  } else {
    a = tg_rect{c.x + w, c.y, lw, h};
    b = tg_rect{c.x, c.y + h, c.w, lh};
  }
  if (a.w > 0 && a.h > 0) cv.free.push_back(a);
  if (b.w > 0 && b.h > 0) cv.free.push_back(b);
  st.refresh_bound(ch.canvas);
  tg_placement pl;
  pl.patch_id = p.patch_id;
  pl.canvas_index = ch.canvas;
  pl.position = tg_rect{c.x, c.y, w, h};
  pl.reserved = 0;
  cv.placed.push_back(Placed{pl, queue_index});
  cv.used += static_cast<int64_t>(w) * h;
}

struct Queued {
  tg_patch_meta meta;
  int32_t src_frame;
};

struct Event {
  tg_invoke_info info;
  std::vector<Queued> patches;    // queue order
  std::vector<Placed> placements; // canvas-major
  std::vector<tg_free_rect> free; // canvas-major, list order
};

}  // namespace

struct tg_batcher {
  tg_canvas_spec spec{};
  Profile prof;
  int max_canvases = 1;
  std::vector<Queued> queue;
  Packing st;
  int64_t t_ddl = 0, t_remain = 0;
  bool has_timer = false;
  int64_t timer_at = 0;
  uint64_t timer_epoch = 0, next_epoch = 1;
  std::vector<Event> events;
  // Optional event log: the records the reference SloScheduler writes
  // (scheduler.hpp:93-99 arrival, 153-159 repack, 173-178 invoke, 186-188
  // timer_set) through EventLog::record (event_log.hpp: nlohmann dump(),
  // keys sorted, plus "policy"), one JSON line each, byte for byte.
  bool log_on = false;
  std::string policy, log;

  static const char* trigger_name(tg_trigger t) {
    return t == TG_TRIGGER_DEADLINE_TIMER ? "deadline_timer"
           : t == TG_TRIGGER_INFEASIBLE_ARRIVAL ? "infeasible_arrival"
                                                : "memory_cap";
  }
  void logf(const char* fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    log += buf;
  }
  void log_arrival(const tg_patch_meta& p, int64_t now) {
    if (!log_on) return;
    logf("{\"deadline_us\":%lld,\"event\":\"arrival\",\"h\":%d,\"patch\":%llu,\"policy\":\"%s\","
         "\"t_us\":%lld,\"w\":%d}\n",
         static_cast<long long>(p.deadline_us), p.rect.h,
         static_cast<unsigned long long>(p.patch_id), policy.c_str(), static_cast<long long>(now),
         p.rect.w);
  }
  void log_repack(int64_t now, size_t n, int k, int64_t slack, int64_t remain) {
    if (!log_on) return;
    logf("{\"canvases\":%d,\"event\":\"repack\",\"patches\":%zu,\"policy\":\"%s\",\"slack_us\":%lld,"
         "\"t_remain_us\":%lld,\"t_us\":%lld}\n",
         k, n, policy.c_str(), static_cast<long long>(slack), static_cast<long long>(remain),
         static_cast<long long>(now));
  }
  void log_timer() {
    if (!log_on) return;
    logf("{\"epoch\":%llu,\"event\":\"timer_set\",\"fire_at_us\":%lld,\"policy\":\"%s\"}\n",
         static_cast<unsigned long long>(timer_epoch), static_cast<long long>(timer_at),
         policy.c_str());
  }
  void log_invoke(const Event& ev) {
    if (!log_on) return;
    logf("{\"event\":\"invoke\",\"k\":%d,\"patches\":[", ev.info.batch_size);
    for (size_t i = 0; i < ev.patches.size(); ++i)
      logf(i ? ",%llu" : "%llu", static_cast<unsigned long long>(ev.patches[i].meta.patch_id));
    logf("],\"policy\":\"%s\",\"slack_us\":%lld,\"t_us\":%lld,\"trigger\":\"%s\"}\n",
         policy.c_str(), static_cast<long long>(ev.info.estimated_slack_us),
         static_cast<long long>(ev.info.fire_time_us),
         trigger_name(static_cast<tg_trigger>(ev.info.trigger)));
  }

  void reset() {
    queue.clear();
    st = Packing{};
    has_timer = false;
    t_ddl = 0;
    t_remain = 0;
  }

  void make_event(int64_t now, tg_trigger trig) {
    Event ev;
    ev.info.fire_time_us = now;
    ev.info.batch_size = static_cast<int32_t>(st.canvases.size());
    ev.info.trigger = trig;
    ev.info.estimated_slack_us = prof.slack_us(ev.info.batch_size);
    ev.info.n_patches = static_cast<int32_t>(queue.size());
    ev.patches = queue;
    for (int ci = 0; ci < static_cast<int>(st.canvases.size()); ++ci) {
      const CanvasSt& c = st.canvases[ci];
      for (const Placed& p : c.placed) ev.placements.push_back(p);
      for (int k = 0; k < static_cast<int>(c.free.size()); ++k)
        ev.free.push_back(tg_free_rect{c.free[k], ci, k});
    }
    ev.info.n_free = static_cast<int32_t>(ev.free.size());
    log_invoke(ev);
    events.push_back(std::move(ev));
  }

  tg_status arrival(const tg_patch_meta& p, int32_t src, int64_t now) {
    const int M = spec.width, N = spec.height;
    log_arrival(p, now);
    if (p.rect.w > M || p.rect.h > N)  // stitch.hpp:114-118 (raised inside repack)
      return bfail(TG_ERR_INVALID_ARGUMENT, "patch exceeds canvas (patch %llu, %dx%d)",
                   static_cast<unsigned long long>(p.patch_id), p.rect.w, p.rect.h);
    // tentative repack (scheduler.hpp:101-104) as one incremental placement
    const Choice ch = choose(st, p.rect.w, p.rect.h, M, N);
    const int k = static_cast<int>(st.canvases.size()) + (ch.fi < 0 ? 1 : 0);
    const int64_t ddl = queue.empty() ? p.deadline_us : std::min(t_ddl, p.deadline_us);
    const int64_t remain = ddl - prof.slack_us(k);
    log_repack(now, queue.size() + 1, k, prof.slack_us(k), remain);
    const bool over_cap = k > max_canvases;
    if (over_cap || remain < now) {                      // :106-123
      const tg_trigger trig = over_cap ? TG_TRIGGER_MEMORY_CAP : TG_TRIGGER_INFEASIBLE_ARRIVAL;
      if (!queue.empty()) make_event(now, trig);         // the pre-arrival batch
      reset();
      queue.push_back(Queued{p, src});
      commit(st, choose(st, p.rect.w, p.rect.h, M, N), p, 0, M, N);
      t_ddl = p.deadline_us;
      t_remain = t_ddl - prof.slack_us(1);
      log_repack(now, 1, 1, prof.slack_us(1), t_remain);
      if (t_remain < now) {                              // infeasible even alone
        make_event(now, TG_TRIGGER_INFEASIBLE_ARRIVAL);
        reset();
        return TG_OK;
      }
    } else {
      commit(st, ch, p, static_cast<int>(queue.size()), M, N);
      queue.push_back(Queued{p, src});
      t_ddl = ddl;
      t_remain = remain;
    }
    has_timer = true;                                    // arm_timer :124
    timer_at = t_remain;
    timer_epoch = next_epoch++;
    log_timer();
    return TG_OK;
  }

  void timer(int64_t now, uint64_t epoch) {               // :130-135
    if (!has_timer || timer_epoch != epoch || queue.empty()) return;
    make_event(now, TG_TRIGGER_DEADLINE_TIMER);
    reset();
  }
};

namespace {

tg_status to_job(const tg_gather_job& j, Job* out) {
  const tg_rect& d = j.dst;
  if (d.x < 0 || d.y < 0 || d.w < 1 || d.h < 1 || d.x + d.w > 65535 || d.y + d.h > 65535 ||
      j.src_x < 0 || j.src_y < 0 || j.src_x > 65535 || j.src_y > 65535)
    return bfail(TG_ERR_INVALID_ARGUMENT, "gather job out of the 16-bit coordinate range");
  *out = Job{static_cast<uint16_t>(d.x), static_cast<uint16_t>(d.y), static_cast<uint16_t>(d.w),
             static_cast<uint16_t>(d.h), j.src_frame, static_cast<uint16_t>(j.src_x),
             static_cast<uint16_t>(j.src_y)};
  return TG_OK;
}

}  // namespace

extern "C" {

tg_status tg_stitch_gather(tg_ctx* ctx, const tg_gather_job* jobs, int32_t n_jobs,
                           const int32_t* canvas_job_offsets, int32_t n_canvases,
                           tg_canvas_spec spec, const uint8_t* const* d_frames, int32_t pitch,
                           uint8_t* d_canvases, void* stream) {
  if (!ctx) return bfail(TG_ERR_INVALID_ARGUMENT, "null context");
  if (n_canvases < 0 || n_jobs < 0) return bfail(TG_ERR_INVALID_ARGUMENT, "negative counts");
  if (pitch % 16) return bfail(TG_ERR_INVALID_ARGUMENT, "pitch must be a multiple of 16");
  std::vector<Job> hj(static_cast<size_t>(n_jobs));
  std::vector<uint2> ranges(static_cast<size_t>(n_canvases));
  for (int c = 0; c < n_canvases; ++c) {
    const int a = canvas_job_offsets[c], b = canvas_job_offsets[c + 1];
    if (a < 0 || b < a || b > n_jobs) return bfail(TG_ERR_INVALID_ARGUMENT, "bad job offsets");
    for (int i = a; i < b; ++i) {
      const tg_status s = to_job(jobs[i], &hj[i]);
      if (s) return s;
    }
    std::sort(hj.begin() + a, hj.begin() + b, [](const Job& x, const Job& y) {
      return x.dx != y.dx ? x.dx < y.dx : x.dy < y.dy;
    });
    ranges[c] = make_uint2(static_cast<uint32_t>(a), static_cast<uint32_t>(b - a));
  }
  return tg_internal_run_gather(ctx, hj.data(), n_jobs, ranges.data(), n_canvases, spec, d_frames,
                                pitch, d_canvases, stream);
}

tg_status tg_profile_slack_us(const tg_profile_entry* entries, int32_t n, int32_t k,
                              int64_t* slack_us) {
  Profile p;
  const tg_status s = Profile::make(entries, n, &p);
  if (s) return s;
  if (k < 1) return bfail(TG_ERR_INVALID_ARGUMENT, "invalid batch size");
  *slack_us = p.slack_us(k);
  return TG_OK;
}

tg_status tg_max_canvases_per_batch(double gpu_memory_gb, double model_size_gb,
                                    double vram_per_canvas_gb, int32_t* k) {
  if (vram_per_canvas_gb <= 0) return bfail(TG_ERR_INVALID_ARGUMENT, "vram per canvas must be positive");
  const double head_room = gpu_memory_gb - model_size_gb;
  const int v = static_cast<int>(std::floor(head_room / vram_per_canvas_gb + 1e-9));
  if (v < 1) return bfail(TG_ERR_INVALID_ARGUMENT, "cannot fit one canvas in GPU memory");
  *k = v;
  return TG_OK;
}

tg_status tg_transmission_schedule(const tg_patch_meta* patches, int32_t n, double bandwidth_mbps,
                                   int64_t* arrival_us) {
  if (!(bandwidth_mbps > 0.0)) return bfail(TG_ERR_INVALID_ARGUMENT, "bandwidth must be positive");
  int64_t link_free_at = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t start = std::max(patches[i].generation_time_us, link_free_at);
    const double bits = static_cast<double>(patches[i].size_bytes) * 8.0;
    const int64_t arrival = start + std::llround(bits / bandwidth_mbps);  // Mbps == bits/us
    arrival_us[i] = arrival;
    link_free_at = arrival;
  }
  return TG_OK;
}

tg_status tg_batcher_create(tg_canvas_spec spec, const tg_profile_entry* entries, int32_t n_entries,
                            int32_t max_canvases, tg_batcher** out) {
  *out = nullptr;
  if (n_entries > 0 && entries == nullptr)
    return bfail(TG_ERR_INVALID_ARGUMENT, "scheduler needs a latency profile");
  if (n_entries <= 0) return bfail(TG_ERR_INVALID_ARGUMENT, "scheduler needs a latency profile");
  if (max_canvases < 1) return bfail(TG_ERR_INVALID_ARGUMENT, "max canvases must be >= 1");
  if (spec.width < 1 || spec.height < 1 || spec.width > 65535 || spec.height > 65535)
    return bfail(TG_ERR_INVALID_ARGUMENT, "canvas dimensions must be in [1, 65535]");
  tg_batcher* b = new tg_batcher();
  const tg_status s = Profile::make(entries, n_entries, &b->prof);
  if (s) {
    delete b;
    return s;
  }
  b->spec = spec;
  b->max_canvases = max_canvases;
  *out = b;
  return TG_OK;
}

void tg_batcher_destroy(tg_batcher* b) { delete b; }

tg_status tg_batcher_set_log(tg_batcher* b, const char* policy) {
  b->log_on = policy != nullptr;
  b->policy = policy ? policy : "";
  b->log.clear();
  return TG_OK;
}

tg_status tg_batcher_take_log(tg_batcher* b, char* out, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(b->log.size());
  if (out == nullptr) return TG_OK;  // size query
  if (cap < *len) return bfail(TG_ERR_CAPACITY, "log buffer too small (%lld < %lld)",
                               static_cast<long long>(cap), static_cast<long long>(*len));
  std::copy(b->log.begin(), b->log.end(), out);
  b->log.clear();
  return TG_OK;
}

tg_status tg_batcher_on_patch_arrival(tg_batcher* b, const tg_patch_meta* patch, int32_t src_frame,
                                      int64_t now_us, int32_t* n_events) {
  b->events.clear();
  const tg_status s = b->arrival(*patch, src_frame, now_us);
  *n_events = static_cast<int32_t>(b->events.size());
  return s;
}

tg_status tg_batcher_on_timer(tg_batcher* b, int64_t now_us, uint64_t epoch, int32_t* n_events) {
  b->events.clear();
  b->timer(now_us, epoch);
  *n_events = static_cast<int32_t>(b->events.size());
  return TG_OK;
}

tg_status tg_batcher_pending_timer(tg_batcher* b, int32_t* has_timer, int64_t* fire_at_us,
                                   uint64_t* epoch) {
  *has_timer = b->has_timer ? 1 : 0;
  *fire_at_us = b->has_timer ? b->timer_at : 0;
  *epoch = b->has_timer ? b->timer_epoch : 0;
  return TG_OK;
}

tg_status tg_batcher_status(tg_batcher* b, int32_t* queue_len, int32_t* canvases,
                            int64_t* earliest_deadline_us, int64_t* remaining_time_us) {
  *queue_len = static_cast<int32_t>(b->queue.size());
  *canvases = static_cast<int32_t>(b->st.canvases.size());
  *earliest_deadline_us = b->t_ddl;
  *remaining_time_us = b->t_remain;
  return TG_OK;
}

tg_status tg_batcher_current(tg_batcher* b, tg_invoke_info* info, tg_patch_meta* queue,
                             tg_placement* placements, tg_free_rect* free_rects) {
  tg_invoke_info in{};
  in.batch_size = static_cast<int32_t>(b->st.canvases.size());
  in.n_patches = static_cast<int32_t>(b->queue.size());
  in.estimated_slack_us = in.batch_size > 0 ? b->prof.slack_us(in.batch_size) : 0;
  int32_t nf = 0, np = 0;
  for (int ci = 0; ci < in.batch_size; ++ci) {
    const CanvasSt& c = b->st.canvases[ci];
    for (const Placed& p : c.placed) {
      if (placements) placements[np] = p.pl;
      ++np;
    }
    for (int k = 0; k < static_cast<int>(c.free.size()); ++k) {
      if (free_rects) free_rects[nf] = tg_free_rect{c.free[k], ci, k};
      ++nf;
    }
  }
  in.n_free = nf;
  if (queue)
    for (size_t k = 0; k < b->queue.size(); ++k) queue[k] = b->queue[k].meta;
  if (info) *info = in;
  return TG_OK;
}

tg_status tg_batcher_event(tg_batcher* b, int32_t i, tg_invoke_info* info, uint64_t* patch_ids,
                           tg_placement* placements, tg_free_rect* free_rects) {
  if (i < 0 || i >= static_cast<int32_t>(b->events.size()))
    return bfail(TG_ERR_OUT_OF_RANGE, "event index out of range");
  const Event& ev = b->events[i];
  if (info) *info = ev.info;
  if (patch_ids)
    for (size_t k = 0; k < ev.patches.size(); ++k) patch_ids[k] = ev.patches[k].meta.patch_id;
  if (placements)
    for (size_t k = 0; k < ev.placements.size(); ++k) placements[k] = ev.placements[k].pl;
  if (free_rects) std::copy(ev.free.begin(), ev.free.end(), free_rects);
  return TG_OK;
}

}  // extern "C"

namespace {
// Appends one event's canvases to the flat plan: placements pull from their
// patch's frame, final free rects zero-fill; jobs x-sorted per canvas.
tg_status append_event_plan(const Event& ev, std::vector<Job>& jobs, std::vector<uint2>& ranges) {
  const int nc = ev.info.batch_size;
  std::vector<std::vector<Job>> per(static_cast<size_t>(nc));
  for (const Placed& p : ev.placements) {
    const Queued& q = ev.patches[p.queue_index];
    Job j;
    const tg_status s =
        to_job(tg_gather_job{p.pl.position, q.src_frame, q.meta.rect.x, q.meta.rect.y}, &j);
    if (s) return s;
    if (q.src_frame < 0)
      return bfail(TG_ERR_INVALID_ARGUMENT, "patch %llu has no source frame",
                   static_cast<unsigned long long>(q.meta.patch_id));
    per[p.pl.canvas_index].push_back(j);
  }
  for (const tg_free_rect& f : ev.free) {
    Job j;
    const tg_status s = to_job(tg_gather_job{f.rect, -1, 0, 0}, &j);
    if (s) return s;
    per[f.canvas_index].push_back(j);
  }
  for (auto& v : per) {
    std::sort(v.begin(), v.end(), [](const Job& x, const Job& y) {
      return x.dx != y.dx ? x.dx < y.dx : x.dy < y.dy;
    });
    ranges.push_back(make_uint2(static_cast<uint32_t>(jobs.size()), static_cast<uint32_t>(v.size())));
    jobs.insert(jobs.end(), v.begin(), v.end());
  }
  return TG_OK;
}
}  // namespace

extern "C" {

tg_status tg_batcher_gather(tg_ctx* ctx, tg_batcher* b, int32_t i, const uint8_t* const* d_frames,
                            int32_t pitch, uint8_t* d_canvases, void* stream) {
  if (i < 0 || i >= static_cast<int32_t>(b->events.size()))
    return bfail(TG_ERR_OUT_OF_RANGE, "event index out of range");
  std::vector<Job> jobs;
  std::vector<uint2> ranges;
  const tg_status s = append_event_plan(b->events[i], jobs, ranges);
  if (s) return s;
  return tg_internal_run_gather(ctx, jobs.data(), static_cast<int32_t>(jobs.size()), ranges.data(),
                                static_cast<int32_t>(ranges.size()), b->spec, d_frames, pitch,
                                d_canvases, stream);
}

tg_status tg_batcher_gather_events(tg_ctx* ctx, tg_batcher* b, int32_t first, int32_t stride,
                                   const uint8_t* const* d_frames, int32_t pitch,
                                   uint8_t* d_canvases, int64_t canvas_cap, int64_t* n_canvases,
                                   void* stream) {
  *n_canvases = 0;
  if (stride < 1 || first < 0 || first >= stride)
    return bfail(TG_ERR_INVALID_ARGUMENT, "event subset needs 0 <= first < stride");
  std::vector<Job> jobs;
  std::vector<uint2> ranges;
  for (size_t e = static_cast<size_t>(first); e < b->events.size(); e += static_cast<size_t>(stride)) {
    const tg_status s = append_event_plan(b->events[e], jobs, ranges);
    if (s) return s;
  }
  *n_canvases = static_cast<int64_t>(ranges.size());
  if (static_cast<int64_t>(ranges.size()) > canvas_cap)
    return bfail(TG_ERR_CAPACITY, "canvas capacity exceeded (%lld canvases > %lld)",
                 static_cast<long long>(ranges.size()), static_cast<long long>(canvas_cap));
  return tg_internal_run_gather(ctx, jobs.data(), static_cast<int32_t>(jobs.size()), ranges.data(),
                                static_cast<int32_t>(ranges.size()), b->spec, d_frames, pitch,
                                d_canvases, stream);
}

tg_status tg_batcher_gather_all(tg_ctx* ctx, tg_batcher* b, const uint8_t* const* d_frames,
                                int32_t pitch, uint8_t* d_canvases, int64_t canvas_cap,
                                int64_t* n_canvases, void* stream) {
  return tg_batcher_gather_events(ctx, b, 0, 1, d_frames, pitch, d_canvases, canvas_cap,
                                  n_canvases, stream);
}

tg_status tg_batcher_replay(tg_batcher* b, const tg_patch_meta* patches, const int32_t* src_frames,
                            const int64_t* arrival_us, int32_t n, int32_t* n_events) {
  // sim.hpp:334-342 (arrival seqs first, scene-major), 392-400 (timer pushed
  // when its epoch is new), 425-458 (heap by (t, seq)).  The reference's heap
  // is replayed without one: arrivals hold seqs 0..n-1, so they pop in
  // (t, index) order -- one sort -- and precede any timer at equal t (timer
  // seqs are >= n).  Only the newest timer can fire: an older epoch's timer
  // pops as a no-op (scheduler.hpp:130-135), so a single pending (t, epoch)
  // stands in for the heap's timer entries.
  std::vector<std::pair<int64_t, int32_t>> order(static_cast<size_t>(n));
  bool sorted = true;
  for (int i = 0; i < n; ++i) {
    order[i] = {arrival_us[i], i};
    if (i && order[i] < order[i - 1]) sorted = false;
  }
  if (!sorted) std::sort(order.begin(), order.end());
  std::vector<Event> all;
  bool timer_pending = false;
  int64_t timer_t = 0;
  uint64_t timer_ep = 0, pushed_epoch = 0;
  size_t next = 0;
  while (next < order.size() || timer_pending) {
    b->events.clear();
    if (next < order.size() && (!timer_pending || order[next].first <= timer_t)) {
      const int i = order[next++].second;
      const tg_status s = b->arrival(patches[i], src_frames ? src_frames[i] : -1, arrival_us[i]);
      if (s) return s;
      if (b->has_timer && b->timer_epoch != pushed_epoch) {
        timer_pending = true;
        timer_t = b->timer_at;
        timer_ep = b->timer_epoch;
        pushed_epoch = b->timer_epoch;
      }
    } else {
      timer_pending = false;
      b->timer(timer_t, timer_ep);
    }
    for (auto& e : b->events) all.push_back(std::move(e));
  }
  b->events = std::move(all);
  *n_events = static_cast<int32_t>(b->events.size());
  if (!b->queue.empty()) return bfail(TG_ERR_INVALID_ARGUMENT, "scheduler queue not drained");
  return TG_OK;
}

tg_status tg_batcher_replay_links(tg_batcher* b, int32_t n_cams, const int32_t* cam_offsets,
                                  const tg_patch_meta* patches, const int32_t* src_frames,
                                  double bandwidth_mbps, int32_t per_camera_link,
                                  int64_t* arrival_us_out, int32_t* n_events) {
  const int n = cam_offsets[n_cams];
  std::vector<int64_t> arrival(static_cast<size_t>(n));
  if (per_camera_link) {
    for (int c = 0; c < n_cams; ++c) {
      const int a = cam_offsets[c], e = cam_offsets[c + 1];
      const tg_status s = tg_transmission_schedule(patches + a, e - a, bandwidth_mbps, arrival.data() + a);
      if (s) return s;
    }
  } else {  // one shared link: (generation time, patch id) order (sim.hpp:280-289)
    std::vector<int> order(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) {
      return std::tie(patches[x].generation_time_us, patches[x].patch_id) <
             std::tie(patches[y].generation_time_us, patches[y].patch_id);
    });
    std::vector<tg_patch_meta> merged(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) merged[i] = patches[order[i]];
    std::vector<int64_t> arr(static_cast<size_t>(n));
    const tg_status s = tg_transmission_schedule(merged.data(), n, bandwidth_mbps, arr.data());
    if (s) return s;
    for (int i = 0; i < n; ++i) arrival[order[i]] = arr[i];
  }
  if (arrival_us_out) std::copy(arrival.begin(), arrival.end(), arrival_us_out);
  return tg_batcher_replay(b, patches, src_frames, arrival.data(), n, n_events);
}

}  // extern "C"

extern "C" {

tg_status tg_descriptors_compact(const tg_patch_meta* patches, const int32_t* n_patches,
                                 const uint8_t* admitted, int32_t zones, const int32_t* cameras,
                                 int32_t n_cams, int32_t frames_per_camera, tg_descriptor* out,
                                 int64_t cap, int64_t* n_out) {
  *n_out = 0;
  if (zones < 1 || n_cams < 0 || frames_per_camera < 0)
    return bfail(TG_ERR_INVALID_ARGUMENT, "bad descriptor layout");
  int64_t k = 0;
  const int64_t F = static_cast<int64_t>(n_cams) * frames_per_camera;
  for (int64_t f = 0; f < F; ++f) {
    const int np = n_patches[f];
    if (np < 0 || np > zones) return bfail(TG_ERR_INVALID_ARGUMENT, "bad patch count");
    if (k + np > cap) return bfail(TG_ERR_CAPACITY, "descriptor capacity exceeded");
    const int cam = cameras[f / frames_per_camera];
    const int fr = static_cast<int>(f % frames_per_camera);
    for (int j = 0; j < np; ++j) {
      tg_descriptor& d = out[k++];
      d.patch = patches[f * zones + j];
      d.camera = cam;
      d.frame = fr;
      d.admitted = admitted[f * zones + j] ? 1 : 0;
      d.pad = 0;
    }
  }
  *n_out = k;
  return TG_OK;
}

tg_status tg_batcher_schedule(tg_batcher* b, const tg_descriptor* desc, int64_t n,
                              const int32_t* cameras, int32_t n_cams, int32_t frames_per_camera,
                              double bandwidth_mbps, int32_t per_camera_link,
                              tg_patch_meta* admitted_out, int32_t* src_frames_out,
                              int64_t* arrival_us_out, int64_t* n_admitted, int32_t* n_events) {
  *n_events = 0;
  if (n_admitted) *n_admitted = 0;
  if (n < 0 || n_cams < 0 || frames_per_camera < 0)
    return bfail(TG_ERR_INVALID_ARGUMENT, "bad descriptor counts");
  int32_t max_cam = -1;
  for (int k = 0; k < n_cams; ++k) {
    if (cameras[k] < 0) return bfail(TG_ERR_INVALID_ARGUMENT, "negative camera id");
    max_cam = std::max(max_cam, cameras[k]);
  }
  std::vector<int32_t> slot_of(static_cast<size_t>(max_cam) + 1, -1);
  for (int k = 0; k < n_cams; ++k) slot_of[cameras[k]] = k;
  std::vector<tg_patch_meta> adm;
  std::vector<int32_t> src;
  std::vector<int32_t> count(static_cast<size_t>(n_cams), 0);
  adm.reserve(static_cast<size_t>(n));
  src.reserve(static_cast<size_t>(n));
  int last_slot = 0;
  for (int64_t i = 0; i < n; ++i) {
    const tg_descriptor& d = desc[i];
    const int slot = (d.camera >= 0 && d.camera <= max_cam) ? slot_of[d.camera] : -1;
    if (slot < 0) continue;  // another shard's camera: it only takes its id
    if (slot < last_slot)
      return bfail(TG_ERR_INVALID_ARGUMENT,
                   "descriptor %lld: camera %d out of the camera order", static_cast<long long>(i),
                   d.camera);
    last_slot = slot;
    if (d.frame < 0 || d.frame >= frames_per_camera)
      return bfail(TG_ERR_INVALID_ARGUMENT, "descriptor %lld: frame %d out of range",
                   static_cast<long long>(i), d.frame);
    if (!d.admitted) continue;
    tg_patch_meta p = d.patch;
    p.patch_id = static_cast<uint64_t>(i);
    adm.push_back(p);
    src.push_back(slot * (frames_per_camera + 1) + d.frame + 1);
    ++count[slot];
  }
  std::vector<int32_t> offs(static_cast<size_t>(n_cams) + 1, 0);
  for (int k = 0; k < n_cams; ++k) offs[k + 1] = offs[k] + count[k];
  const int32_t na = static_cast<int32_t>(adm.size());
  if (n_admitted) *n_admitted = na;
  if (admitted_out) std::copy(adm.begin(), adm.end(), admitted_out);
  if (src_frames_out) std::copy(src.begin(), src.end(), src_frames_out);
  return tg_batcher_replay_links(b, n_cams, offs.data(), adm.data(), src.data(), bandwidth_mbps,
                                 per_camera_link, arrival_us_out, n_events);
}

}  // extern "C"
