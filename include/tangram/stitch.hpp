// tangram/stitch.hpp -- drop-in for the reference's patch-stitching header
// (stitch.hpp:30-208).  stitch_all() runs Alg. 2's BSSF + guillotine solver
// on the B200 (tg_stitch_all) with bit-identical placements and free lists
// in the reference's list order; the result helpers are host value code.
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/partition.hpp"

namespace tangram {

struct CanvasSpec {
  int width = 1024;
  int height = 1024;
  double vram_per_canvas_gb = 1.0;
  [[nodiscard]] std::int64_t surface_area() const { return std::int64_t{width} * height; }
};

struct Placement {
  std::uint64_t patch_id = 0;
  int canvas_index = 0;
  Rect position;
};

struct CanvasState {
  std::vector<Placement> placements;
  std::vector<Rect> free_rects;
  std::int64_t used_area = 0;
};

struct StitchResult {
  CanvasSpec spec;
  std::vector<CanvasState> canvases;
  std::map<std::uint64_t, Placement> placement_index;
  [[nodiscard]] int canvas_count() const { return static_cast<int>(canvases.size()); }
  [[nodiscard]] bool empty() const { return canvases.empty(); }
};

inline StitchResult stitch_all(std::span<const PatchMeta> queue, const CanvasSpec& spec) {
  StitchResult res;
  res.spec = spec;
  if (queue.empty()) return res;
  const std::size_t n = queue.size();
  std::vector<tg_patch_meta> q;
  q.reserve(n);
  for (const PatchMeta& p : queue) q.push_back(gpu::to_c(p));
  std::vector<tg_placement> pl(n);
  std::vector<tg_free_rect> fr(2 * n + 1);
  int32_t nc = 0, nf = 0;
  gpu::check(tg_stitch_all(gpu::Context::get(), q.data(), static_cast<int32_t>(n),
                           tg_canvas_spec{spec.width, spec.height, spec.vram_per_canvas_gb},
                           pl.data(), &nc, fr.data(), static_cast<int32_t>(fr.size()), &nf));
  res.canvases.resize(static_cast<std::size_t>(nc));
  for (const tg_placement& p : pl) {
    const Placement placed{p.patch_id, p.canvas_index, gpu::from_c(p.position)};
    CanvasState& c = res.canvases[static_cast<std::size_t>(p.canvas_index)];
    c.placements.push_back(placed);
    c.used_area += area(placed.position);
    res.placement_index[placed.patch_id] = placed;
  }
  for (int i = 0; i < nf; ++i)
    res.canvases[static_cast<std::size_t>(fr[i].canvas_index)].free_rects.push_back(
        gpu::from_c(fr[i].rect));
  return res;
}

inline std::vector<double> canvas_efficiency(const StitchResult& result) {
  const double s = static_cast<double>(result.spec.surface_area());
  std::vector<double> eff;
  eff.reserve(result.canvases.size());
  for (const CanvasState& c : result.canvases) eff.push_back(static_cast<double>(c.used_area) / s);
  return eff;
}

inline std::string dump_layout(const StitchResult& result) {
  const std::vector<double> eff = canvas_efficiency(result);
  std::string text;
  char buf[160];
  for (int ci = 0; ci < result.canvas_count(); ++ci) {
    std::snprintf(buf, sizeof(buf), "canvas %d (%dx%d) efficiency=%.4f\n", ci, result.spec.width,
                  result.spec.height, eff[static_cast<std::size_t>(ci)]);
    text += buf;
    for (const Placement& p : result.canvases[static_cast<std::size_t>(ci)].placements) {
      std::snprintf(buf, sizeof(buf), "  patch %llu at (%d,%d) %dx%d\n",
                    static_cast<unsigned long long>(p.patch_id), p.position.x, p.position.y,
                    p.position.w, p.position.h);
      text += buf;
    }
  }
  return text;
}

inline StitchResult extract_canvas(const StitchResult& result, int canvas_index) {
  if (canvas_index < 0 || canvas_index >= result.canvas_count())
    throw std::out_of_range("canvas index out of range");
  StitchResult one;
  one.spec = result.spec;
  one.canvases.push_back(result.canvases[static_cast<std::size_t>(canvas_index)]);
  for (Placement& p : one.canvases.front().placements) {
    p.canvas_index = 0;
    one.placement_index[p.patch_id] = p;
  }
  return one;
}

inline StitchResult concat_stitches(std::span<const StitchResult> parts) {
  StitchResult all;
  if (!parts.empty()) all.spec = parts.front().spec;
  for (const StitchResult& part : parts) {
    const int shift = all.canvas_count();
    for (CanvasState c : part.canvases) {
      for (Placement& p : c.placements) {
        p.canvas_index += shift;
        all.placement_index[p.patch_id] = p;
      }
      all.canvases.push_back(std::move(c));
    }
  }
  return all;
}

}  // namespace tangram
