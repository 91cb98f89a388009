// tangram/scheduler.hpp -- drop-in for the reference's SLO-aware batching
// invoker (scheduler.hpp:29-215, Alg. 2).  Same types (InvokeTrigger,
// InvokeEvent, TimerHandle), constructor, exceptions and member functions;
// the state machine is the C ABI's tg_batcher (csrc/batcher.cu): identical
// decisions, timer epochs, triggers and stitch results, with an incremental
// repack (stitch_all is prefix-consistent) instead of a full
// stitch_all() of the queue per arrival.  With an EventLog the batcher's
// arrival / repack / invoke / timer_set lines are written to it,
// byte-identical to the reference's.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

#include "tangram/event_log.hpp"
#include "tangram/latency.hpp"
#include "tangram/stitch.hpp"

namespace tangram {

enum class InvokeTrigger {
  deadline_timer,
  infeasible_arrival,
  memory_cap,
};

inline const char* to_string(InvokeTrigger t) {
  switch (t) {
    case InvokeTrigger::deadline_timer: return "deadline_timer";
    case InvokeTrigger::infeasible_arrival: return "infeasible_arrival";
    case InvokeTrigger::memory_cap: return "memory_cap";
  }
  return "?";
}

struct InvokeEvent {
  Micros fire_time_us = 0;
  StitchResult stitch;
  std::vector<std::uint64_t> patch_ids;
  int batch_size = 0;
  Micros estimated_slack_us = 0;
  InvokeTrigger trigger = InvokeTrigger::deadline_timer;
};

struct TimerHandle {
  Micros fire_at_us = 0;
  std::uint64_t epoch = 0;
};

class SloScheduler {
 public:
  SloScheduler(CanvasSpec spec, const LatencyProfile* profile, int max_canvases,
               EventLog* log = nullptr)
      : spec_(spec), log_(log) {
    if (profile == nullptr) throw std::invalid_argument("scheduler needs a latency profile");
    if (max_canvases < 1) throw std::invalid_argument("max canvases must be >= 1");
    gpu::check(tg_batcher_create(tg_canvas_spec{spec.width, spec.height, spec.vram_per_canvas_gb},
                                 profile->c_entries(), profile->c_count(), max_canvases, &b_));
    if (log_ != nullptr && log_->enabled()) gpu::check(tg_batcher_set_log(b_, log_->policy().c_str()));
  }
  ~SloScheduler() { tg_batcher_destroy(b_); }
  SloScheduler(const SloScheduler&) = delete;
  SloScheduler& operator=(const SloScheduler&) = delete;
  SloScheduler(SloScheduler&& o) noexcept { *this = std::move(o); }
  SloScheduler& operator=(SloScheduler&& o) noexcept {
    std::swap(spec_, o.spec_);
    std::swap(log_, o.log_);
    std::swap(b_, o.b_);
    std::swap(fresh_, o.fresh_);
    queue_ = std::move(o.queue_);
    current_ = std::move(o.current_);
    previous_ = std::move(o.previous_);
    return *this;
  }

  // Zero, one or (flush + solo-infeasible dispatch) two invocations, in firing order.
  std::vector<InvokeEvent> on_patch_arrival(const PatchMeta& patch, Micros now) {
    const StitchResult before = current_stitch();
    int32_t n = 0;
    const tg_patch_meta p = gpu::to_c(patch);
    const tg_status s = tg_batcher_on_patch_arrival(b_, &p, -1, now, &n);
    flush_log();
    fresh_ = false;
    gpu::check(s);
    std::vector<InvokeEvent> out = events(n);
    // scheduler.hpp:101-121: previous_ holds the pre-arrival packing unless
    // this arrival flushed (then it is cleared)
    previous_ = out.empty() ? before : StitchResult{};
    return out;
  }

  // Fires the current batch; superseded timers (older epochs) are no-ops.
  std::optional<InvokeEvent> on_timer(Micros now, std::uint64_t epoch) {
    int32_t n = 0;
    gpu::check(tg_batcher_on_timer(b_, now, epoch, &n));
    flush_log();
    if (n == 0) return std::nullopt;
    fresh_ = false;
    previous_ = StitchResult{};
    return events(n).front();
  }

  std::optional<TimerHandle> pending_timer() const {
    int32_t has = 0;
    int64_t at = 0;
    uint64_t ep = 0;
    gpu::check(tg_batcher_pending_timer(b_, &has, &at, &ep));
    if (!has) return std::nullopt;
    return TimerHandle{at, ep};
  }
  bool idle() const { return status().q == 0; }
  const std::vector<PatchMeta>& queue() const {
    refresh();
    return queue_;
  }
  const StitchResult& current_stitch() const {
    refresh();
    return current_;
  }
  const StitchResult& previous_stitch() const { return previous_; }
  Micros earliest_deadline_us() const { return status().ddl; }
  Micros remaining_time_us() const { return status().remain; }

 private:
  struct Status {
    int32_t q, k;
    int64_t ddl, remain;
  };
  Status status() const {
    Status st{};
    gpu::check(tg_batcher_status(b_, &st.q, &st.k, &st.ddl, &st.remain));
    return st;
  }

  static StitchResult to_result(const CanvasSpec& spec, int canvases, const tg_placement* pl,
                                int n_pl, const tg_free_rect* fr, int n_fr) {
    StitchResult r;
    r.spec = spec;
    r.canvases.resize(static_cast<std::size_t>(canvases));
    for (int i = 0; i < n_pl; ++i) {
      const Placement p{pl[i].patch_id, pl[i].canvas_index, gpu::from_c(pl[i].position)};
      CanvasState& c = r.canvases[static_cast<std::size_t>(p.canvas_index)];
      c.placements.push_back(p);
      c.used_area += area(p.position);
      r.placement_index[p.patch_id] = p;
    }
    for (int i = 0; i < n_fr; ++i)
      r.canvases[static_cast<std::size_t>(fr[i].canvas_index)].free_rects.push_back(gpu::from_c(fr[i].rect));
    return r;
  }

  std::vector<InvokeEvent> events(int32_t n) const {
    std::vector<InvokeEvent> out;
    for (int32_t i = 0; i < n; ++i) {
      tg_invoke_info info{};
      gpu::check(tg_batcher_event(b_, i, &info, nullptr, nullptr, nullptr));
      std::vector<uint64_t> ids(static_cast<std::size_t>(info.n_patches));
      std::vector<tg_placement> pl(static_cast<std::size_t>(info.n_patches));
      std::vector<tg_free_rect> fr(static_cast<std::size_t>(info.n_free));
      gpu::check(tg_batcher_event(b_, i, &info, ids.data(), pl.data(), fr.data()));
      InvokeEvent e;
      e.fire_time_us = info.fire_time_us;
      e.stitch = to_result(spec_, info.batch_size, pl.data(), info.n_patches, fr.data(), info.n_free);
      e.patch_ids = std::move(ids);
      e.batch_size = info.batch_size;
      e.estimated_slack_us = info.estimated_slack_us;
      e.trigger = static_cast<InvokeTrigger>(info.trigger);
      out.push_back(std::move(e));
    }
    return out;
  }

  // the live queue and packing, fetched once per state change
  void refresh() const {
    if (fresh_) return;
    tg_invoke_info info{};
    gpu::check(tg_batcher_current(b_, &info, nullptr, nullptr, nullptr));
    std::vector<tg_patch_meta> q(static_cast<std::size_t>(info.n_patches));
    std::vector<tg_placement> pl(static_cast<std::size_t>(info.n_patches));
    std::vector<tg_free_rect> fr(static_cast<std::size_t>(info.n_free));
    gpu::check(tg_batcher_current(b_, &info, q.data(), pl.data(), fr.data()));
    queue_.clear();
    for (const tg_patch_meta& m : q) queue_.push_back(gpu::from_c(m));
    current_ = info.batch_size > 0
                   ? to_result(spec_, info.batch_size, pl.data(), info.n_patches, fr.data(), info.n_free)
                   : StitchResult{};
    fresh_ = true;
  }

  void flush_log() {
    if (log_ == nullptr || !log_->enabled()) return;
    int64_t len = 0;
    gpu::check(tg_batcher_take_log(b_, nullptr, 0, &len));
    if (len == 0) return;
    std::string buf(static_cast<std::size_t>(len), '\0');
    gpu::check(tg_batcher_take_log(b_, buf.data(), len, &len));
    log_->write_lines(buf);
  }

  CanvasSpec spec_;
  EventLog* log_ = nullptr;
  tg_batcher* b_ = nullptr;
  mutable bool fresh_ = false;
  mutable std::vector<PatchMeta> queue_;
  mutable StitchResult current_;
  StitchResult previous_;
};

}  // namespace tangram
