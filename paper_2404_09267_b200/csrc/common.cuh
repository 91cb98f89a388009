// common.cuh -- shared device helpers for the sm_100a Tangram kernels.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tangram_gpu.h"

namespace tg {

constexpr int kCell = TG_CELL_SIZE;   // 16x16-pixel patch-grid cells
constexpr int kMaxZones = 64;         // zones per partitioner chunk / fast planner variant
constexpr int kMaxPlanZones = 256;    // X*Y supported by the fused per-frame planner
constexpr int kMaxRadius = 8;         // dilation radius bound (K1b register window)

// Device-side error latch (first error wins), read back at sync points.
struct DevError {
  int code;      // tg_status
  int kind;      // which check fired (see api.cu: error_message)
  long long a, b, c, d;
};

enum ErrKind : int {
  kErrNone = 0,
  kErrRoiOutside = 1,      // a = roi index, b = frame slot
  kErrPatchOversize = 2,   // a = patch id, b = w, c = h
  kErrRoiCapacity = 3,     // a = frame, b = rois found, c = cap
  kErrCanvasCapacity = 4,  // a = total canvases, b = cap
  kErrFreeCapacity = 5,    // a = queue
  kErrDescCapacity = 6,    // a = patches, b = cap
};

__device__ __forceinline__ void raise_error(DevError* e, int code, int kind, long long a,
                                            long long b = 0, long long c = 0, long long d = 0) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->kind = kind;
    e->a = a;
    e->b = b;
    e->c = c;
    e->d = d;
    __threadfence();
  }
}

// Gather job: one rectangle of canvas bytes.  src_frame >= 0 copies from
// that frame of the batch at (sx, sy); src_frame < 0 zero-fills (a final
// guillotine free rect; sx|sy<<16 then holds its insertion seq).
struct Job {
  uint16_t dx, dy, w, h;
  int32_t src_frame;
  uint16_t sx, sy;
};
static_assert(sizeof(Job) == 16, "job is 16 bytes");

// Free rect used by the BSSF planner (smem or global).
struct FreeRect {
  int x, y, w, h, canvas, seq;
};

// ---- PTX wrappers: mbarrier + bulk async copy (TMA bulk engine) ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Wait with a suspend-time hint: the warp sleeps in the barrier unit until
// the phase completes (or the hint expires) instead of spinning on issue
// slots its producer needs.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}

// Global -> shared bulk copy completing on an mbarrier (UBLKCP in SASS).
// dst, src and bytes must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- L2 residency hints ------------------------------------------------------
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Bulk global -> shared copy with an L2 policy on the source lines.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void st_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}

// Warp min over unsigned 64-bit keys (two REDUX ops).
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long k) {
  const unsigned hi = static_cast<unsigned>(k >> 32);
  const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
  const unsigned lo = (hi == mhi) ? static_cast<unsigned>(k) : 0xffffffffu;
  const unsigned mlo = __reduce_min_sync(0xffffffffu, lo);
  return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ---- once-only launch setup (host) -------------------------------------------
// Launchers run every step, so the runtime calls that only configure a kernel
// (dynamic smem opt-in, occupancy) are made once per device and kernel, and
// tuning overrides are read from the environment once per process.
constexpr int kMaxDevices = 64;

// Unset (or unparsable): -1.  Read once; later calls return the cached value.
struct EnvInt {
  const char* name;
  std::atomic<int> state{0};  // 0 unread, 1 read
  int value = -1;
  int get() {
    if (state.load(std::memory_order_acquire) == 0) {
      const char* e = std::getenv(name);
      value = e ? std::atoi(e) : -1;
      state.store(1, std::memory_order_release);
    }
    return value;
  }
};

// Per-device high-water mark of the dynamic smem a kernel was opted into.
struct SmemOptIn {
  std::atomic<int> bytes[kMaxDevices] = {};
  template <class K>
  cudaError_t ensure(K* kernel, int smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < kMaxDevices && bytes[dev].load(std::memory_order_relaxed) >= smem)
      return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && dev >= 0 && dev < kMaxDevices) {
      int cur = bytes[dev].load(std::memory_order_relaxed);
      while (cur < smem && !bytes[dev].compare_exchange_weak(cur, smem)) {
      }
    }
    return e;
  }
};

}  // namespace tg
