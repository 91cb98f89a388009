// k_gather.cu -- K5: batched canvas writer (the paper's
// invoke(canvases) input).
//
// Every canvas is exactly tiled by its placements plus its final guillotine
// free rects, so the job list writes every canvas byte
// exactly once: patch pixels for placements, zeros for free rects.  A
// persistent grid walks (canvas, 32-row band) units -- equal 96 KB of output
// per unit at 1024x1024 RGB -- whose count the scan kernel left in device
// memory, so no host round trip sits between planning and gathering.
// Within a unit each warp copies whole rect rows: destination-aligned
// 16-byte chunks, sources realigned with funnel shifts from two aligned
// 16-byte loads, byte stores only for the (at most two) chunks a row shares
// with its neighbours.
#include "kernels.cuh"

namespace tg {

constexpr int kGatherThreads = 256;
constexpr int kGatherBand = 32;
constexpr int kGatherUnroll = 4;

__device__ __forceinline__ uint4 ldg128(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// 16 bytes starting at an arbitrary address p (all 32 covering bytes lie in
// the same 16B-aligned row).
__device__ __forceinline__ uint4 load16_unaligned(const uint8_t* p) {
  const uintptr_t ip = reinterpret_cast<uintptr_t>(p);
  const uint8_t* q = reinterpret_cast<const uint8_t*>(ip & ~static_cast<uintptr_t>(15));
  const int s = static_cast<int>(ip & 15);
  const uint4 v0 = ldg128(q);
  if (s == 0) return v0;
  const uint4 v1 = ldg128(q + 16);
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  const int sh = 8 * (s & 3);
  uint4 r;
  switch (s >> 2) {
    case 0:
      r = make_uint4(__funnelshift_r(w[0], w[1], sh), __funnelshift_r(w[1], w[2], sh),
                     __funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh));
      break;
    case 1:
      r = make_uint4(__funnelshift_r(w[1], w[2], sh), __funnelshift_r(w[2], w[3], sh),
                     __funnelshift_r(w[3], w[4], sh), __funnelshift_r(w[4], w[5], sh));
      break;
    case 2:
      r = make_uint4(__funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh),
                     __funnelshift_r(w[4], w[5], sh), __funnelshift_r(w[5], w[6], sh));
      break;
    default:
      r = make_uint4(__funnelshift_r(w[3], w[4], sh), __funnelshift_r(w[4], w[5], sh),
                     __funnelshift_r(w[5], w[6], sh), __funnelshift_r(w[6], w[7], sh));
      break;
  }
  return r;
}

// Copies len bytes src -> dst (or zero-fills when src == nullptr).
__device__ __forceinline__ void copy_row(uint8_t* dst, const uint8_t* src, int len, int lane) {
  const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + static_cast<uintptr_t>(len);
  const uintptr_t a0 = d0 & ~static_cast<uintptr_t>(15);
  const int nch = static_cast<int>((((d1 + 15) & ~static_cast<uintptr_t>(15)) - a0) >> 4);
  for (int base = lane; base < nch; base += 32 * kGatherUnroll) {
    uint4 v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const int c = base + 32 * u;
      v[u] = make_uint4(0, 0, 0, 0);
      const uintptr_t A = a0 + 16 * static_cast<uintptr_t>(c);
      if (c < nch && src && A >= d0 && A + 16 <= d1) v[u] = load16_unaligned(src + (A - d0));
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const int c = base + 32 * u;
      if (c >= nch) break;
      const uintptr_t A = a0 + 16 * static_cast<uintptr_t>(c);
      if (A >= d0 && A + 16 <= d1) {
        *reinterpret_cast<uint4*>(A) = v[u];
      } else {
        const uintptr_t lo = A > d0 ? A : d0, hi = (A + 16) < d1 ? (A + 16) : d1;
        for (uintptr_t b = lo; b < hi; ++b)
          *reinterpret_cast<uint8_t*>(b) = src ? __ldg(src + (b - d0)) : 0;
      }
    }
  }
}

__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const GatherArgs a) {
  __shared__ Job sj[3 * kMaxZones];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = kGatherThreads / 32;
  const int nunits = *a.units;
  const size_t canvas_bytes = static_cast<size_t>(a.M) * a.N * 3;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int k = u / a.nbands, b = u - k * a.nbands;
    const uint32_t packed = a.canvas_map[k];
    const int f = static_cast<int>(packed >> 6), c = static_cast<int>(packed & 63u);
    const uint32_t cj = a.canvas_jobs[static_cast<size_t>(f) * a.zones + c];
    const int start = static_cast<int>(cj & 0xffffu), cnt = static_cast<int>(cj >> 16);
    __syncthreads();
    for (int i = tid; i < cnt; i += kGatherThreads)
      sj[i] = a.jobs[static_cast<size_t>(f) * a.job_cap + start + i];
    __syncthreads();
    const int b0 = b * kGatherBand, b1 = min(a.N, b0 + kGatherBand);
    uint8_t* canvas = a.out + static_cast<size_t>(k) * canvas_bytes;
    int seg = 0;
    for (int j = 0; j < cnt; ++j) {
      const Job J = sj[j];
      const int r0 = max(static_cast<int>(J.dy), b0);
      const int r1 = min(static_cast<int>(J.dy) + static_cast<int>(J.h), b1);
      if (r1 <= r0) continue;
      // rows r with (seg + r - r0) % nwarps == warp
      int first = r0 + ((warp - seg) % nwarps + nwarps) % nwarps;
      const uint8_t* sbase =
          J.src_frame >= 0 ? a.frames[J.src_frame] + static_cast<size_t>(J.sx) * 3 : nullptr;
      for (int r = first; r < r1; r += nwarps) {
        const uint8_t* src =
            sbase ? sbase + static_cast<size_t>(J.sy + (r - J.dy)) * a.pitch : nullptr;
        copy_row(canvas + (static_cast<size_t>(r) * a.M + J.dx) * 3, src, 3 * J.w, lane);
      }
      seg += r1 - r0;
    }
  }
}

cudaError_t launch_gather(const GatherArgs& a, int sms, cudaStream_t stream) {
  gather_kernel<<<sms * 4, kGatherThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

int gather_bands(int N) { return ceil_div(N, kGatherBand); }

}  // namespace tg
