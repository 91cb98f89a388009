// scheduler_test.cpp -- the C++ drop-in batcher (include/tangram/
// scheduler.hpp, latency.hpp, cost.hpp, rng.hpp, event_log.hpp) exercised
// with the expectations of the reference's own unit tests
// (proj/tests/scheduler_test.cpp:56-320: 370 ms / 300 ms timers, memory cap,
// infeasible arrival, solo dispatch, flush + solo, zero remaining time,
// stale timers, constructor validation, every patch fires exactly once,
// byte-identical event-log replay, trigger names), plus the latency and
// cost KATs the scheduler depends on.
//
// The same source compiles against the reference headers
// (-I/root/reference/proj/include): tests/test_cpp_scheduler.py runs both
// builds and requires identical output, event logs included.  Host-only: the
// batcher never touches the GPU.
#include <cstdio>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/cost.hpp"
#include "tangram/rng.hpp"
#include "tangram/scheduler.hpp"

using namespace tangram;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)

template <class E, class F>
static std::string expect_throw(F f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (...) {
    return "<wrong exception type>";
  }
  return "<no exception>";
}

// slack(1) = 130 ms, slack(2) = 200 ms
static LatencyProfile kat_profile() {
  return LatencyProfile::from_entries(100, 100, {{1, 100.0, 10.0}, {2, 170.0, 10.0}});
}

static CanvasSpec canvas100() {
  CanvasSpec c;
  c.width = 100;
  c.height = 100;
  return c;
}

static PatchMeta whole(std::uint64_t id, Micros gen, Micros slo) {
  PatchMeta p;
  p.patch_id = id;
  p.source_frame_id = id;
  p.rect = Rect{0, 0, 100, 100};
  p.generation_time_us = gen;
  p.slo_us = slo;
  p.deadline_us = gen + slo;
  p.size_bytes = 15000;
  return p;
}

static std::vector<std::uint64_t> ids(std::initializer_list<std::uint64_t> v) { return v; }

static void kat_timers() {
  const LatencyProfile prof = kat_profile();
  {  // one arrival arms the deadline timer at deadline - slack(1)
    SloScheduler s(canvas100(), &prof, 2);
    CHECK(s.on_patch_arrival(whole(1, 0, 500'000), 0).empty());
    CHECK(!s.idle());
    CHECK(s.earliest_deadline_us() == 500'000 && s.remaining_time_us() == 370'000);
    CHECK(s.pending_timer().has_value() && s.pending_timer()->fire_at_us == 370'000);
    const auto ev = s.on_timer(370'000, s.pending_timer()->epoch);
    CHECK(ev.has_value() && ev->fire_time_us == 370'000 && ev->batch_size == 1);
    CHECK(ev->patch_ids == ids({1}) && ev->estimated_slack_us == 130'000);
    CHECK(ev->trigger == InvokeTrigger::deadline_timer);
    CHECK(s.idle() && !s.pending_timer().has_value());
  }
  {  // a second arrival re-arms with slack(2); the stale timer is a no-op
    SloScheduler s(canvas100(), &prof, 2);
    s.on_patch_arrival(whole(1, 0, 500'000), 0);
    const std::uint64_t stale = s.pending_timer()->epoch;
    CHECK(s.on_patch_arrival(whole(2, 100'000, 500'000), 100'000).empty());
    CHECK(s.queue().size() == 2u && s.current_stitch().canvas_count() == 2);
    CHECK(s.earliest_deadline_us() == 500'000 && s.remaining_time_us() == 300'000);
    CHECK(s.pending_timer()->fire_at_us == 300'000);
    CHECK(!s.on_timer(370'000, stale).has_value());
    CHECK(s.queue().size() == 2u);
    const auto ev = s.on_timer(300'000, s.pending_timer()->epoch);
    CHECK(ev.has_value() && ev->batch_size == 2 && ev->patch_ids == ids({1, 2}));
    CHECK(ev->estimated_slack_us == 200'000);
  }
}

static void kat_flushes() {
  const LatencyProfile prof = kat_profile();
  {  // memory cap: a third full canvas flushes the pair
    SloScheduler s(canvas100(), &prof, 2);
    s.on_patch_arrival(whole(1, 0, 500'000), 0);
    s.on_patch_arrival(whole(2, 100'000, 500'000), 100'000);
    const auto evs = s.on_patch_arrival(whole(3, 250'000, 500'000), 250'000);
    CHECK(evs.size() == 1u);
    if (evs.size() == 1u) {
      CHECK(evs[0].trigger == InvokeTrigger::memory_cap && evs[0].fire_time_us == 250'000);
      CHECK(evs[0].batch_size == 2 && evs[0].patch_ids == ids({1, 2}));
      CHECK(evs[0].estimated_slack_us == 200'000);
    }
    CHECK(s.queue().size() == 1u && s.queue()[0].patch_id == 3u);
    CHECK(s.earliest_deadline_us() == 750'000 && s.remaining_time_us() == 620'000);
    CHECK(s.pending_timer()->fire_at_us == 620'000);
    const auto ev = s.on_timer(620'000, s.pending_timer()->epoch);
    CHECK(ev.has_value() && ev->patch_ids == ids({3}) && s.idle());
  }
  {  // infeasible arrival flushes the pair, the newcomer requeues
    SloScheduler s(canvas100(), &prof, 4);
    PatchMeta a = whole(1, 0, 500'000);
    a.rect = Rect{0, 0, 50, 100};
    PatchMeta b = whole(2, 200'000, 260'000);
    b.rect = Rect{50, 0, 50, 100};
    s.on_patch_arrival(a, 0);
    CHECK(s.on_patch_arrival(b, 200'000).empty());
    CHECK(s.current_stitch().canvas_count() == 1 && s.remaining_time_us() == 330'000);
    CHECK(s.previous_stitch().canvas_count() == 1);  // the packing before b joined
    PatchMeta c = whole(3, 340'000, 140'000);
    const auto evs = s.on_patch_arrival(c, 340'000);
    CHECK(evs.size() == 1u);
    if (evs.size() == 1u) {
      CHECK(evs[0].trigger == InvokeTrigger::infeasible_arrival);
      CHECK(evs[0].patch_ids == ids({1, 2}) && evs[0].batch_size == 1);
      CHECK(evs[0].stitch.canvases.size() == 1u && evs[0].stitch.canvases[0].placements.size() == 2u);
    }
    CHECK(s.previous_stitch().empty());
    CHECK(s.queue().size() == 1u && s.remaining_time_us() == 350'000);
    CHECK(s.pending_timer()->fire_at_us == 350'000);
  }
  {  // unmeetable alone: dispatched solo at once
    SloScheduler s(canvas100(), &prof, 2);
    const auto evs = s.on_patch_arrival(whole(1, 0, 120'000), 0);
    CHECK(evs.size() == 1u);
    if (evs.size() == 1u)
      CHECK(evs[0].trigger == InvokeTrigger::infeasible_arrival && evs[0].fire_time_us == 0 &&
            evs[0].batch_size == 1 && evs[0].patch_ids == ids({1}));
    CHECK(s.idle() && !s.pending_timer().has_value());
  }
  {  // flush and solo dispatch in one arrival
    SloScheduler s(canvas100(), &prof, 2);
    s.on_patch_arrival(whole(1, 0, 500'000), 0);
    const auto evs = s.on_patch_arrival(whole(2, 300'000, 120'000), 300'000);
    CHECK(evs.size() == 2u);
    if (evs.size() == 2u) {
      CHECK(evs[0].trigger == InvokeTrigger::infeasible_arrival && evs[0].patch_ids == ids({1}));
      CHECK(evs[0].fire_time_us == 300'000 && evs[1].fire_time_us == 300'000);
      CHECK(evs[1].trigger == InvokeTrigger::infeasible_arrival && evs[1].patch_ids == ids({2}));
    }
    CHECK(s.idle());
  }
  {  // deadline == slack(1): feasible, the timer fires at once
    SloScheduler s(canvas100(), &prof, 2);
    CHECK(s.on_patch_arrival(whole(1, 0, 130'000), 0).empty());
    CHECK(s.pending_timer().has_value() && s.pending_timer()->fire_at_us == 0);
    const auto ev = s.on_timer(0, s.pending_timer()->epoch);
    CHECK(ev.has_value() && ev->trigger == InvokeTrigger::deadline_timer);
  }
  {  // a timer after the reset is ignored
    SloScheduler s(canvas100(), &prof, 2);
    s.on_patch_arrival(whole(1, 0, 500'000), 0);
    const std::uint64_t ep = s.pending_timer()->epoch;
    CHECK(s.on_timer(370'000, ep).has_value());
    CHECK(!s.on_timer(370'000, ep).has_value());
  }
}

static void kat_validation() {
  const LatencyProfile prof = kat_profile();
  CHECK(expect_throw<std::invalid_argument>([] { SloScheduler(canvas100(), nullptr, 2); }) ==
        "scheduler needs a latency profile");
  CHECK(expect_throw<std::invalid_argument>([&] { SloScheduler(canvas100(), &prof, 0); }) ==
        "max canvases must be >= 1");
  CHECK(std::string(to_string(InvokeTrigger::deadline_timer)) == "deadline_timer");
  CHECK(std::string(to_string(InvokeTrigger::infeasible_arrival)) == "infeasible_arrival");
  CHECK(std::string(to_string(InvokeTrigger::memory_cap)) == "memory_cap");
  // latency.hpp: slack = mu + 3 sigma, interpolated / extrapolated, clamped at 0
  CHECK(prof.slack_us(1) == 130'000 && prof.slack_us(2) == 200'000 && prof.slack_us(3) == 270'000);
  CHECK(prof.slack_ms(2) == 200.0 && prof.mu_ms(3) == 240.0 && prof.sigma_ms(4) == 10.0);
  const LatencyProfile down = LatencyProfile::from_entries(64, 64, {{4, 40.0, 0.0}, {2, 50.0, 0.0}});
  CHECK(down.slack_us(8) == 20'000 && down.slack_us(20) == 0 && down.slack_us(1) == 55'000);
  CHECK(down.entries()[0].batch_size == 2 && down.max_profiled_batch() == 4);
  std::vector<std::string> warn;
  LatencyProfile::from_entries(64, 64, {{1, 50.0, 1.0}, {2, 40.0, 1.0}}, &warn);
  CHECK(warn.size() == 1u && warn[0] == "profile mu decreases from k=1 to k=2");
  CHECK(expect_throw<std::invalid_argument>([] { LatencyProfile::from_entries(1, 1, {}); }) ==
        "latency profile has no entries");
  CHECK(expect_throw<std::invalid_argument>(
            [] { LatencyProfile::from_entries(1, 1, {{1, 1.0, 0.0}, {1, 2.0, 0.0}}); }) ==
        "duplicate profile entry for batch size 1");
  CHECK(expect_throw<std::invalid_argument>([] { LatencyProfile::from_entries(1, 1, {{0, 1.0, 0.0}}); }) ==
        "profile entry with batch size < 1");
  CHECK(expect_throw<std::invalid_argument>([] { LatencyProfile::from_entries(1, 1, {{1, 0.0, 0.0}}); }) ==
        "profile entry with non-positive mu");
  CHECK(expect_throw<std::invalid_argument>([] { LatencyProfile::from_entries(1, 1, {{1, 1.0, -1.0}}); }) ==
        "profile entry with negative sigma");
  CHECK(expect_throw<std::invalid_argument>([&] { (void)prof.slack_us(0); }) == "invalid batch size");
  // cost.hpp:107-115
  FunctionConfig fc;
  CHECK(max_canvases_per_batch(fc, CanvasSpec{}) == 4);
  fc.gpu_memory_gb = 80.0;
  fc.model_size_gb = 4.0;
  CHECK(max_canvases_per_batch(fc, CanvasSpec{}) == 76);
  fc.gpu_memory_gb = 2.5;
  fc.model_size_gb = 2.0;
  CHECK(expect_throw<std::invalid_argument>([&] { max_canvases_per_batch(fc, CanvasSpec{}); }) ==
        "cannot fit one canvas in GPU memory");
  CanvasSpec zero;
  zero.vram_per_canvas_gb = 0.0;
  CHECK(expect_throw<std::invalid_argument>([&] { max_canvases_per_batch(FunctionConfig{}, zero); }) ==
        "vram per canvas must be positive");
}

// The simulator's driving rule: deliver the pending timer whenever it
// precedes the next arrival.
static std::vector<InvokeEvent> drive(SloScheduler& s, const std::vector<PatchMeta>& patches) {
  std::vector<InvokeEvent> all;
  auto fire_due = [&](Micros until, bool all_timers) {
    while (s.pending_timer().has_value() &&
           (all_timers || s.pending_timer()->fire_at_us <= until)) {
      const TimerHandle h = *s.pending_timer();
      auto ev = s.on_timer(h.fire_at_us, h.epoch);
      if (ev.has_value()) all.push_back(std::move(*ev));
    }
  };
  for (const PatchMeta& p : patches) {
    fire_due(p.generation_time_us, false);
    for (auto& e : s.on_patch_arrival(p, p.generation_time_us)) all.push_back(std::move(e));
  }
  fire_due(0, true);
  return all;
}

static std::vector<PatchMeta> random_stream(std::uint64_t seed, int n) {
  Rng rng(seed);
  std::vector<PatchMeta> out;
  Micros t = 0;
  for (int i = 0; i < n; ++i) {
    t += rng.uniform_int(0, 120'000);
    PatchMeta p;
    p.patch_id = static_cast<std::uint64_t>(i + 1);
    p.source_frame_id = static_cast<std::uint64_t>(i);
    const int w = static_cast<int>(rng.uniform_int(10, 100));
    const int h = static_cast<int>(rng.uniform_int(10, 100));
    p.rect = Rect{0, 0, w, h};
    p.generation_time_us = t;
    p.slo_us = rng.uniform_int(125'000, 2'000'000);
    p.deadline_us = t + p.slo_us;
    p.size_bytes = static_cast<std::int64_t>(w) * h;
    out.push_back(p);
  }
  return out;
}

// Every patch fires exactly once, batches respect the cap, timers fire at
// the batch's remaining time; each event is also printed (compared between
// the drop-in and reference builds).
static void random_streams() {
  const LatencyProfile prof = kat_profile();
  for (std::uint64_t seed = 1; seed <= 20; ++seed) {
    SloScheduler s(canvas100(), &prof, 3);
    const auto patches = random_stream(seed, 200);
    const auto events = drive(s, patches);
    std::map<std::uint64_t, Micros> ddl;
    for (const PatchMeta& p : patches) ddl[p.patch_id] = p.deadline_us;
    std::set<std::uint64_t> seen;
    Micros last = 0;
    for (const InvokeEvent& e : events) {
      CHECK(e.fire_time_us >= last);
      last = e.fire_time_us;
      CHECK(e.batch_size >= 1 && e.batch_size <= 3);
      CHECK(e.estimated_slack_us == prof.slack_us(e.batch_size));
      Micros min_ddl = std::numeric_limits<Micros>::max();
      for (std::uint64_t id : e.patch_ids) {
        CHECK(seen.insert(id).second);
        min_ddl = std::min(min_ddl, ddl.at(id));
      }
      if (e.trigger == InvokeTrigger::deadline_timer) CHECK(e.fire_time_us == min_ddl - e.estimated_slack_us);
      std::printf("seed %llu t %lld %s k %d slack %lld ids", static_cast<unsigned long long>(seed),
                  static_cast<long long>(e.fire_time_us), to_string(e.trigger), e.batch_size,
                  static_cast<long long>(e.estimated_slack_us));
      for (std::uint64_t id : e.patch_ids) std::printf(" %llu", static_cast<unsigned long long>(id));
      for (const CanvasState& c : e.stitch.canvases) {
        for (const Placement& p : c.placements)
          std::printf(" p%llu@%d:%d,%d", static_cast<unsigned long long>(p.patch_id), p.canvas_index,
                      p.position.x, p.position.y);
        for (const Rect& r : c.free_rects) std::printf(" f%d,%d,%d,%d", r.x, r.y, r.w, r.h);
      }
      std::printf("\n");
    }
    CHECK(seen.size() == patches.size());
    CHECK(s.idle());
  }
}

// Two runs of one stream write byte-identical event logs (printed for the
// comparison with the reference build).
static void event_log_replay() {
  const LatencyProfile prof = kat_profile();
  const auto patches = random_stream(99, 120);
  std::string first;
  for (int run = 0; run < 2; ++run) {
    std::ostringstream out;
    EventLog log(&out, "tangram");
    SloScheduler s(canvas100(), &prof, 3, &log);
    drive(s, patches);
    if (run == 0) {
      first = out.str();
      CHECK(first.find("\"event\":\"invoke\"") != std::string::npos);
      CHECK(first.find("\"event\":\"timer_set\"") != std::string::npos);
    } else {
      CHECK(out.str() == first);
    }
  }
  std::printf("%s", first.c_str());
}

int main() {
  kat_timers();
  kat_flushes();
  kat_validation();
  random_streams();
  event_log_replay();
  std::printf("scheduler_test: %s\n", g_fail ? "FAILURES" : "ALL PASS");
  return g_fail ? 1 : 0;
}
