// k_synth.cu -- synthetic camera frames on the device (fixture source; not
// part of any timed region).  Same frozen pixel spec as the oracle's
// orc_synth_frame: background 96 + h&63, per-frame noise in
// [-3,3], foreground 32 + h&15 on even frames and 224 - h&15 on odd ones,
// inside the frame's generate_trace() rects (trace.hpp:184-231).
#include "kernels.cuh"

namespace tg {

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// grid: (row blocks, frames); each thread writes 4 bytes of one row.
__global__ void __launch_bounds__(256) synth_kernel(const SynthArgs a) {
  const int fi = blockIdx.y;
  const int t = a.t0 + fi;
  const int rowbytes = 3 * a.W;
  const int words_per_row = rowbytes / 4;
  const long long gidx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gidx >= static_cast<long long>(words_per_row) * a.H) return;
  const int y = static_cast<int>(gidx / words_per_row);
  const int j0 = static_cast<int>(gidx - static_cast<long long>(y) * words_per_row) * 4;
  const uint32_t s_bg = static_cast<uint32_t>(a.seed);
  const uint32_t s_fg = hash32(s_bg ^ 0x5bd1e995u);
  const uint32_t tn = hash32(static_cast<uint32_t>(a.seed >> 32) + static_cast<uint32_t>(t));
  const uint32_t tf = s_fg ^ (static_cast<uint32_t>(t) * 0x9E3779B9u);
  const int r0 = t >= 0 ? a.offsets[fi] : 0, r1 = t >= 0 ? a.offsets[fi + 1] : 0;
  uint32_t out = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    const int x = j / 3;
    const uint32_t idx = static_cast<uint32_t>(y) * static_cast<uint32_t>(rowbytes) + static_cast<uint32_t>(j);
    bool fg = false;
    for (int r = r0; r < r1 && !fg; ++r) {
      const tg_rect R = a.rects[r];
      fg = x >= R.x && x < R.x + R.w && y >= R.y && y < R.y + R.h;
    }
    int base;
    if (fg) {
      const int h = static_cast<int>(hash32(idx ^ tf) & 15u);
      base = (t & 1) ? 224 - h : 32 + h;
    } else {
      base = 96 + static_cast<int>(hash32(idx ^ s_bg) & 63u);
    }
    const int n = static_cast<int>(hash32(idx ^ tn) % 7u) - 3;
    const int v = min(255, max(0, base + n));
    out |= static_cast<uint32_t>(v) << (8 * k);
  }
  *reinterpret_cast<uint32_t*>(a.frames[fi] + static_cast<size_t>(y) * a.pitch + j0) = out;
}

cudaError_t launch_synth(const SynthArgs& a, int n_frames, cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  const long long words = static_cast<long long>(3 * a.W / 4) * a.H;
  dim3 grid(static_cast<unsigned>((words + 255) / 256), static_cast<unsigned>(n_frames));
  synth_kernel<<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace tg
