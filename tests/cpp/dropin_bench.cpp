// dropin_bench.cpp -- per-call cost of the C++ drop-in a reference caller
// sees: tangram::partition + tangram::stitch_all once per 4K frame, the way
// the reference's run() loops (sim.hpp:248-250, 319).  The same source
// compiles against the reference headers (CPU) and against include/tangram
// (each call a device round trip through the C ABI); both builds print the
// same placement checksum, then microseconds per frame.
//   tests/cpp/Makefile: dropin_bench (drop-in), dropin_bench_ref (reference)
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tangram/rng.hpp"
#include "tangram/stitch.hpp"

using namespace tangram;

int main(int argc, char** argv) {
  const int frames = argc > 1 ? std::atoi(argv[1]) : 300;
  const int W = 3840, H = 2160;
  // synthetic RoIs: 2..12 per frame, 16..480 px sides, inside the frame
  Rng rng(derive_seed(1000, "dropin-bench"));
  std::vector<std::vector<Rect>> rois(static_cast<std::size_t>(frames));
  for (auto& fr : rois) {
    const int n = static_cast<int>(rng.uniform_int(2, 12));
    for (int i = 0; i < n; ++i) {
      const int w = static_cast<int>(rng.uniform_int(16, 480)), h = static_cast<int>(rng.uniform_int(16, 480));
      fr.push_back(Rect{static_cast<int>(rng.uniform_int(0, W - w)), static_cast<int>(rng.uniform_int(0, H - h)), w, h});
    }
  }
  const PartitionConfig cfg{4, 4};
  const CanvasSpec canvas{};
  auto pass = [&](std::uint64_t* checksum, long long* canvases) {
    std::uint64_t first = 0, sum = 0;
    long long nc = 0;
    for (int f = 0; f < frames; ++f) {
      FrameSpec fs;
      fs.frame_id = static_cast<std::uint64_t>(f);
      fs.width = W;
      fs.height = H;
      fs.generation_time_us = f * 33'333;
      fs.slo_us = 1'000'000;
      const std::vector<PatchMeta> patches = partition(fs, cfg, rois[static_cast<std::size_t>(f)], 1.5, first);
      first += patches.size();
      std::vector<PatchMeta> admitted;  // sim.hpp:262
      for (const PatchMeta& p : patches)
        if (p.rect.w <= canvas.width && p.rect.h <= canvas.height) admitted.push_back(p);
      const StitchResult r = stitch_all(admitted, canvas);
      nc += r.canvas_count();
      for (const auto& [id, pl] : r.placement_index)
        sum = sum * 1000003u + (id * 31u + static_cast<std::uint64_t>(pl.canvas_index) * 7u +
                                static_cast<std::uint64_t>(pl.position.x) * 65537u +
                                static_cast<std::uint64_t>(pl.position.y));
    }
    *checksum = sum;
    *canvases = nc;
  };
  std::uint64_t checksum = 0;
  long long canvases = 0;
  pass(&checksum, &canvases);  // warm-up (first call creates the device context)
  const int reps = 5;
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    pass(&checksum, &canvases);
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    best = us < best ? us : best;
  }
  std::printf("checksum %016llx canvases %lld\n", static_cast<unsigned long long>(checksum), canvases);
  std::printf("per_frame_us %.2f (partition + stitch_all, best of %d passes over %d frames)\n",
              best / frames, reps, frames);
  return 0;
}
