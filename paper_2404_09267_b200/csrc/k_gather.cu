// k_gather.cu -- K5: batched canvas writer (the paper's
// invoke(canvases) input).
//
// Every canvas is exactly tiled by its placements plus its final guillotine
// free rects: each canvas row is a left-to-right
// sequence of intervals, each either a patch's source row or zeros.  A
// persistent grid walks (canvas, 32-row band) units -- 96 KB of output each
// at 1024x1024 RGB -- whose count the scan kernel left in device memory, so
// no host round trip sits between planning and gathering.  A warp owns whole
// canvas rows: it ballots the canvas's x-sorted jobs into the row's interval
// list (shared memory), then every lane writes 16-byte destination-aligned
// chunks; a chunk inside one interval is one or two aligned 16-byte source
// loads realigned with funnel shifts, a chunk straddling intervals is merged
// in registers with byte masks.  Every store is a full 16-byte store except
// at rows that do not start 16-byte aligned (canvas width % 16 != 0).
#include "kernels.cuh"

namespace tg {

constexpr int kGatherThreads = 256;
constexpr int kGatherWarps = kGatherThreads / 32;
constexpr int kGatherBand = 32;
constexpr int kGatherMaxJobs = 192;  // jobs of one canvas held in smem (row-interval path)

struct RowIv {
  int s, e;            // destination byte range within the canvas row
  const uint8_t* src;  // source bytes for s (nullptr: zero fill)
};

__device__ __forceinline__ uint4 ldg128(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// 16 bytes of a window starting at p (any alignment) whose bytes
// [need_lo, need_hi) are readable; aligned blocks that do not intersect the
// needed bytes are not touched, so reads never leave the source row.
__device__ __forceinline__ uint4 window16(const uint8_t* p, int need_lo, int need_hi) {
  const uintptr_t ip = reinterpret_cast<uintptr_t>(p);
  const uint8_t* q = reinterpret_cast<const uint8_t*>(ip & ~static_cast<uintptr_t>(15));
  const int s = static_cast<int>(ip & 15);
  // block 0 covers window bytes [-s, 16-s), block 1 covers [16-s, 32-s)
  const bool use0 = need_lo < 16 - s && need_hi > -s;
  const bool use1 = s != 0 && need_hi > 16 - s;
  const uint4 v0 = use0 ? ldg128(q) : make_uint4(0, 0, 0, 0);
  if (s == 0) return v0;
  const uint4 v1 = use1 ? ldg128(q + 16) : make_uint4(0, 0, 0, 0);
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  const int sh = 8 * (s & 3);
  switch (s >> 2) {
    case 0:
      return make_uint4(__funnelshift_r(w[0], w[1], sh), __funnelshift_r(w[1], w[2], sh),
                        __funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh));
    case 1:
      return make_uint4(__funnelshift_r(w[1], w[2], sh), __funnelshift_r(w[2], w[3], sh),
                        __funnelshift_r(w[3], w[4], sh), __funnelshift_r(w[4], w[5], sh));
    case 2:
      return make_uint4(__funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh),
                        __funnelshift_r(w[4], w[5], sh), __funnelshift_r(w[5], w[6], sh));
    default:
      return make_uint4(__funnelshift_r(w[3], w[4], sh), __funnelshift_r(w[4], w[5], sh),
                        __funnelshift_r(w[5], w[6], sh), __funnelshift_r(w[6], w[7], sh));
  }
}

__device__ __forceinline__ uint32_t byte_mask(int lo, int hi, int word) {
  const int l = min(max(lo - 4 * word, 0), 4), h = min(max(hi - 4 * word, 0), 4);
  return h > l ? ((0xffffffffu >> (32 - 8 * (h - l))) << (8 * l)) : 0u;
}

__device__ __forceinline__ void merge16(uint4& out, const uint4& v, int lo, int hi) {
  const uint32_t m0 = byte_mask(lo, hi, 0), m1 = byte_mask(lo, hi, 1);
  const uint32_t m2 = byte_mask(lo, hi, 2), m3 = byte_mask(lo, hi, 3);
  out.x = (out.x & ~m0) | (v.x & m0);
  out.y = (out.y & ~m1) | (v.y & m1);
  out.z = (out.z & ~m2) | (v.z & m2);
  out.w = (out.w & ~m3) | (v.w & m3);
}

// Writes one canvas row from its interval list (sorted, tiling [0, len)).
__device__ __forceinline__ void write_row(uint8_t* row, int len, const RowIv* iv, int n_iv,
                                          int lane) {
  const uintptr_t rb = reinterpret_cast<uintptr_t>(row);
  const uintptr_t base = rb & ~static_cast<uintptr_t>(15);
  const int lead = static_cast<int>(rb - base);  // bytes of the first chunk before the row
  const int nch = (lead + len + 15) >> 4;
  constexpr int U = 4;  // chunks per lane in flight
  for (int c0 = lane; c0 < nch; c0 += 32 * U) {
    uint4 out[U];
    int kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // phase 1: locate + issue the fast-path loads
      const int c = c0 + 32 * u;
      out[u] = make_uint4(0, 0, 0, 0);
      kk[u] = -1;
      if (c >= nch) continue;
      const int A = 16 * c - lead;
      const int olo = max(A, 0), ohi = min(A + 16, len);
      int lo = 0, hi = n_iv - 1;  // last interval with s <= olo
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (iv[mid].s <= olo) lo = mid;
        else hi = mid - 1;
      }
      const RowIv first = n_iv ? iv[lo] : RowIv{0, len, nullptr};
      if (first.e >= ohi && olo == A && ohi == A + 16) {
        if (first.src) out[u] = window16(first.src + (A - first.s), 0, 16);
      } else {
        kk[u] = lo;  // straddles intervals or the row edge: phase 2
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // phase 2: merge slow chunks, store
      const int c = c0 + 32 * u;
      if (c >= nch) break;
      const int A = 16 * c - lead;
      const int olo = max(A, 0), ohi = min(A + 16, len);
      if (kk[u] >= 0) {
        for (int k = kk[u]; k < n_iv && iv[k].s < ohi; ++k) {
          const RowIv I = iv[k];
          if (!I.src) continue;  // zero bytes: out already zero there
          const int blo = max(olo, I.s) - A, bhi = min(ohi, I.e) - A;
          merge16(out[u], window16(I.src + (A - I.s), blo, bhi), blo, bhi);
        }
      }
      uint8_t* dst = reinterpret_cast<uint8_t*>(base) + 16 * c;
      if (olo == A && ohi == A + 16) {
        *reinterpret_cast<uint4*>(dst) = out[u];
      } else {  // row edge that is not 16-byte aligned: store only the row's bytes
        const uint32_t w[4] = {out[u].x, out[u].y, out[u].z, out[u].w};
        for (int b = olo - A; b < ohi - A; ++b)
          dst[b] = static_cast<uint8_t>(w[b >> 2] >> (8 * (b & 3)));
      }
    }
  }
}

// Fallback for canvases with more jobs than fit the interval path: copy
// rect rows one by one with byte stores at the edges.
__device__ void copy_rect_row(uint8_t* dst, const uint8_t* src, int len, int lane) {
  const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + static_cast<uintptr_t>(len);
  const uintptr_t a0 = d0 & ~static_cast<uintptr_t>(15);
  const int nch = static_cast<int>((((d1 + 15) & ~static_cast<uintptr_t>(15)) - a0) >> 4);
  for (int c = lane; c < nch; c += 32) {
    const uintptr_t A = a0 + 16 * static_cast<uintptr_t>(c);
    if (A >= d0 && A + 16 <= d1) {
      *reinterpret_cast<uint4*>(A) = src ? window16(src + (A - d0), 0, 16) : make_uint4(0, 0, 0, 0);
    } else {
      const uintptr_t lo = A > d0 ? A : d0, hi = (A + 16) < d1 ? (A + 16) : d1;
      for (uintptr_t b = lo; b < hi; ++b)
        *reinterpret_cast<uint8_t*>(b) = src ? __ldg(src + (b - d0)) : 0;
    }
  }
}

__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const GatherArgs a) {
  __shared__ Job sj[kGatherMaxJobs];
  __shared__ RowIv siv[kGatherWarps][kGatherMaxJobs];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nunits = *a.units;
  const size_t canvas_bytes = static_cast<size_t>(a.M) * a.N * 3;
  const int row_len = 3 * a.M;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int k = u / a.nbands, b = u - k * a.nbands;
    const uint32_t packed = a.canvas_map[k];
    const int f = static_cast<int>(packed >> 6), c = static_cast<int>(packed & 63u);
    const uint32_t cj = a.canvas_jobs[static_cast<size_t>(f) * a.zones + c];
    const int start = static_cast<int>(cj & 0xffffu), cnt = static_cast<int>(cj >> 16);
    const Job* gj = a.jobs + static_cast<size_t>(f) * a.job_cap + start;
    const int b0 = b * kGatherBand, b1 = min(a.N, b0 + kGatherBand);
    uint8_t* canvas = a.out + static_cast<size_t>(k) * canvas_bytes;
    if (cnt <= kGatherMaxJobs) {
      __syncthreads();
      for (int i = tid; i < cnt; i += kGatherThreads) sj[i] = gj[i];
      __syncthreads();
      RowIv* iv = siv[warp];
      for (int r = b0 + warp; r < b1; r += kGatherWarps) {
        int n_iv = 0;
        for (int jb = 0; jb < cnt; jb += 32) {
          const int j = jb + lane;
          bool act = false;
          Job J{};
          if (j < cnt) {
            J = sj[j];
            act = r >= J.dy && r < J.dy + J.h;
          }
          const unsigned m = __ballot_sync(0xffffffffu, act);
          if (act) {
            RowIv e;
            e.s = 3 * J.dx;
            e.e = 3 * (J.dx + J.w);
            e.src = J.src_frame >= 0 ? a.frames[J.src_frame] +
                                           static_cast<size_t>(J.sy + (r - J.dy)) * a.pitch +
                                           static_cast<size_t>(J.sx) * 3
                                     : nullptr;
            iv[n_iv + __popc(m & ((1u << lane) - 1u))] = e;
          }
          n_iv += __popc(m);
        }
        __syncwarp();
        write_row(canvas + static_cast<size_t>(r) * row_len, row_len, iv, n_iv, lane);
        __syncwarp();
      }
    } else {
      int seg = 0;
      for (int j = 0; j < cnt; ++j) {
        const Job J = gj[j];
        const int r0 = max(static_cast<int>(J.dy), b0);
        const int r1 = min(static_cast<int>(J.dy) + static_cast<int>(J.h), b1);
        if (r1 <= r0) continue;
        const int first = r0 + ((warp - seg) % kGatherWarps + kGatherWarps) % kGatherWarps;
        const uint8_t* sbase =
            J.src_frame >= 0 ? a.frames[J.src_frame] + static_cast<size_t>(J.sx) * 3 : nullptr;
        for (int r = first; r < r1; r += kGatherWarps) {
          const uint8_t* src =
              sbase ? sbase + static_cast<size_t>(J.sy + (r - J.dy)) * a.pitch : nullptr;
          copy_rect_row(canvas + static_cast<size_t>(r) * row_len + 3 * J.dx, src, 3 * J.w, lane);
        }
        seg += r1 - r0;
      }
    }
  }
}

cudaError_t launch_gather(const GatherArgs& a, int sms, cudaStream_t stream) {
  gather_kernel<<<sms * 4, kGatherThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

int gather_bands(int N) { return ceil_div(N, kGatherBand); }

}  // namespace tg
