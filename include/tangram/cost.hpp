// tangram/cost.hpp -- drop-in for the part of the reference's cost model
// the batcher depends on (cost.hpp:30-46, 107-115): FunctionConfig and
// max_canvases_per_batch, the memory cap on a batch's canvases (Eq. 5),
// computed by the C ABI (tg_max_canvases_per_batch) with the reference's
// messages.  Billing (PricingTable, invocation_cost*, cost.hpp:48-105) is
// serverless accounting, not the frame->canvas path: out of scope (SURVEY §2
// row 8).
#pragma once

#include <stdexcept>

#include "tangram/stitch.hpp"

namespace tangram {

struct FunctionConfig {
  int vcpus = 2;
  double memory_gb = 4.0;
  double gpu_memory_gb = 6.0;
  double model_size_gb = 2.0;
  int concurrency = 1;

  void validate() const {
    if (vcpus < 1 || memory_gb <= 0 || gpu_memory_gb <= 0 || model_size_gb <= 0 || concurrency < 1)
      throw std::invalid_argument("function config fields must be positive");
    if (model_size_gb >= gpu_memory_gb)
      throw std::invalid_argument("model size must be smaller than GPU memory");
  }
};

// floor((gpu_memory - model_size) / vram_per_canvas), at least 1.
inline int max_canvases_per_batch(const FunctionConfig& cfg, const CanvasSpec& spec) {
  int32_t k = 0;
  gpu::check(tg_max_canvases_per_batch(cfg.gpu_memory_gb, cfg.model_size_gb,
                                       spec.vram_per_canvas_gb, &k));
  return k;
}

}  // namespace tangram
