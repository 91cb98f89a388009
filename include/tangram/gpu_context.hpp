// gpu_context.hpp -- plumbing for the C++ drop-in headers: a lazily created
// per-thread device context and the mapping from C-ABI status codes back to
// the exceptions the reference throws (std::invalid_argument,
// std::out_of_range).  Link with -ltangram_gpu (paper_2404_09267_b200/lib).
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "tangram_gpu.h"

namespace tangram::gpu {

[[noreturn]] inline void raise(tg_status s) {
  const std::string msg = tg_last_error();
  switch (s) {
    case TG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case TG_ERR_CAPACITY: throw std::length_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check(tg_status s) {
  if (s != TG_OK) raise(s);
}

// One context per calling thread (a tg_ctx is not thread-safe; the
// reference's free functions are reentrant).
class Context {
 public:
  static tg_ctx* get() {
    thread_local Context c;
    return c.ctx_;
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

 private:
  Context() {
    int32_t dev = 0;
    if (const char* e = std::getenv("TANGRAM_GPU_DEVICE")) dev = std::atoi(e);
    check(tg_ctx_create(dev, &ctx_));
  }
  ~Context() { tg_ctx_destroy(ctx_); }
  tg_ctx* ctx_ = nullptr;
};

}  // namespace tangram::gpu
