// tangram/partition.hpp -- drop-in for the reference's Alg. 1 header
// (partition.hpp:32-143).  Same types, signatures and exceptions; the work
// runs on the B200 through the C ABI (tg_partition / tg_assign_rois).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "tangram/geometry.hpp"
#include "tangram/gpu_context.hpp"

namespace tangram {

// Integer microseconds internally; milliseconds only at file/CLI edges.
using Micros = std::int64_t;

constexpr Micros ms_to_us(double ms) {
  return ms < 0 ? static_cast<Micros>(ms * 1000.0 - 0.5) : static_cast<Micros>(ms * 1000.0 + 0.5);
}
constexpr double us_to_ms(Micros us) { return static_cast<double>(us) / 1000.0; }

struct FrameSpec {
  std::uint64_t frame_id = 0;
  int width = 0;
  int height = 0;
  Micros generation_time_us = 0;
  Micros slo_us = 0;
};

struct PartitionConfig {
  int zones_x = 4;
  int zones_y = 4;
};

struct PatchMeta {
  std::uint64_t patch_id = 0;
  std::uint64_t source_frame_id = 0;
  Rect rect;
  Micros generation_time_us = 0;
  Micros slo_us = 0;
  Micros deadline_us = 0;
  std::int64_t size_bytes = 0;
};

namespace gpu {
inline tg_frame_spec to_c(const FrameSpec& f) {
  return tg_frame_spec{f.frame_id, f.width, f.height, f.generation_time_us, f.slo_us};
}
inline tg_rect to_c(const Rect& r) { return tg_rect{r.x, r.y, r.w, r.h}; }
inline Rect from_c(const tg_rect& r) { return Rect{r.x, r.y, r.w, r.h}; }
inline tg_patch_meta to_c(const PatchMeta& p) {
  return tg_patch_meta{p.patch_id, p.source_frame_id, to_c(p.rect), p.generation_time_us,
                       p.slo_us, p.deadline_us, p.size_bytes};
}
inline PatchMeta from_c(const tg_patch_meta& p) {
  return PatchMeta{p.patch_id, p.source_frame_id, from_c(p.rect), p.generation_time_us,
                   p.slo_us, p.deadline_us, p.size_bytes};
}
}  // namespace gpu

inline std::vector<Rect> make_zones(const FrameSpec& frame, const PartitionConfig& cfg) {
  const long long n = static_cast<long long>(cfg.zones_x) * cfg.zones_y;
  std::vector<tg_rect> z(n > 0 ? static_cast<std::size_t>(n) : 1);
  const tg_frame_spec fs = gpu::to_c(frame);
  gpu::check(tg_make_zones(&fs, tg_partition_config{cfg.zones_x, cfg.zones_y}, z.data(),
                           static_cast<int32_t>(z.size())));
  std::vector<Rect> out;
  out.reserve(static_cast<std::size_t>(n));
  for (long long i = 0; i < n; ++i) out.push_back(gpu::from_c(z[static_cast<std::size_t>(i)]));
  return out;
}

inline std::vector<std::vector<int>> assign_rois(std::span<const Rect> rois,
                                                 std::span<const Rect> zones) {
  std::vector<tg_rect> r, z;
  for (const Rect& x : rois) r.push_back(gpu::to_c(x));
  for (const Rect& x : zones) z.push_back(gpu::to_c(x));
  std::vector<int32_t> zone_of(rois.size() + 1);
  gpu::check(tg_assign_rois(gpu::Context::get(), r.data(), static_cast<int32_t>(r.size()),
                            z.data(), static_cast<int32_t>(z.size()), zone_of.data()));
  std::vector<std::vector<int>> lists(zones.size());
  for (std::size_t i = 0; i < rois.size(); ++i) lists[zone_of[i]].push_back(static_cast<int>(i));
  return lists;
}

inline std::vector<PatchMeta> partition(const FrameSpec& frame, const PartitionConfig& cfg,
                                        std::span<const Rect> rois, double bytes_per_pixel,
                                        std::uint64_t first_patch_id = 0) {
  std::vector<tg_rect> r;
  r.reserve(rois.size());
  for (const Rect& x : rois) r.push_back(gpu::to_c(x));
  const int cap = cfg.zones_x > 0 && cfg.zones_y > 0 ? cfg.zones_x * cfg.zones_y : 1;
  std::vector<tg_patch_meta> out(static_cast<std::size_t>(cap));
  int32_t n = 0;
  const tg_frame_spec fs = gpu::to_c(frame);
  gpu::check(tg_partition(gpu::Context::get(), &fs, tg_partition_config{cfg.zones_x, cfg.zones_y},
                          r.data(), static_cast<int32_t>(r.size()), bytes_per_pixel,
                          first_patch_id, out.data(), cap, &n));
  std::vector<PatchMeta> patches;
  patches.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) patches.push_back(gpu::from_c(out[static_cast<std::size_t>(i)]));
  return patches;
}

}  // namespace tangram
