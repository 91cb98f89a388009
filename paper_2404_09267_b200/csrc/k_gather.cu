// k_gather.cu -- K5: batched canvas writer (the paper's
// invoke(canvases) input).
//
// Every canvas is exactly tiled by its placements plus its final guillotine
// free rects: each canvas row is a left-to-right
// sequence of intervals, each either a patch's source row or zeros, and the
// sequence only changes at rows where some rect starts or ends.  A
// persistent grid walks (canvas, 256-row band) units whose count the scan
// kernel left in device memory (no host round trip between planning and
// gathering).  Each warp owns 32 contiguous rows of a band.  For a run of
// rows with the same interval set it plans once -- per lane and 16-byte
// destination chunk: zero, single-interval copy (aligned source block +
// funnel-shift amount, row-invariant because pitches are multiples of 16),
// or a boundary chunk that needs a byte-mask merge -- and then streams the
// rows: one or two aligned 16-byte loads, shifts and one full 16-byte store
// per chunk.  Canvases whose rows are not 16-byte aligned (width % 16 != 0)
// or that hold more rects than the interval path caches take a per-rect
// fallback with byte stores at the edges.
#include "kernels.cuh"

namespace tg {

#ifndef TG_GATHER_PLAN_CHUNKS
#define TG_GATHER_PLAN_CHUNKS 6
#endif
#ifndef TG_GATHER_MIN_BLOCKS
#define TG_GATHER_MIN_BLOCKS 2
#endif
#ifndef TG_GATHER_BAND
#define TG_GATHER_BAND 256
#endif

constexpr int kGatherThreads = 256;
constexpr int kGatherWarps = kGatherThreads / 32;
constexpr int kGatherBand = TG_GATHER_BAND;                // rows per unit
constexpr int kPlanChunks = TG_GATHER_PLAN_CHUNKS;         // chunks per lane per segment
constexpr int kSegChunks = 32 * kPlanChunks;               // 3 KB (one 1024-px row) per segment
constexpr int kGatherMaxJobs = 192;                        // rects of one canvas cached in smem

struct RowIv {
  int s, e;          // destination bytes [s, e) of the row
  int zero, pad;     // zero fill (a free rect)
  uintptr_t base;    // source address of dst byte x in row r: base + r * pitch + x
};

__device__ __forceinline__ uint4 ldg128(uintptr_t p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// Plain (weak) global store: __stcg would emit STG.STRONG.GPU.
__device__ __forceinline__ void stg128(uintptr_t p, const uint4& v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Bytes [s, s+16) of the 32-byte pair (v0, v1); branch-free (selects +
// funnel shifts) so a row's loads can all be issued before any realign.
__device__ __forceinline__ uint4 realign(const uint4& v0, const uint4& v1, int s) {
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  const int q = s >> 2, sh = 8 * (s & 3);
  uint32_t p[5];  // p[j] = w[j + q]
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const uint32_t lo = (q & 1) ? w[j + 1] : w[j];
    const uint32_t hi = (q & 1) ? w[j + 3] : w[j + 2];
    p[j] = (q & 2) ? hi : lo;
  }
  return make_uint4(__funnelshift_r(p[0], p[1], sh), __funnelshift_r(p[1], p[2], sh),
                    __funnelshift_r(p[2], p[3], sh), __funnelshift_r(p[3], p[4], sh));
}

// 16 bytes of a window starting at p whose bytes [need_lo, need_hi) are
// readable; aligned blocks not intersecting them are never touched, so reads
// stay inside the source row.
__device__ __forceinline__ uint4 window16(uintptr_t p, int need_lo, int need_hi) {
  const uintptr_t q = p & ~static_cast<uintptr_t>(15);
  const int s = static_cast<int>(p & 15);
  const bool use0 = need_lo < 16 - s && need_hi > -s;
  const bool use1 = s != 0 && need_hi > 16 - s;
  const uint4 z = make_uint4(0, 0, 0, 0);
  const uint4 v0 = use0 ? ldg128(q) : z;
  if (s == 0) return v0;
  return realign(v0, use1 ? ldg128(q + 16) : z, s);
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

// Fallback: copy one rect row with byte stores at unaligned edges.
__device__ void copy_rect_row(uint8_t* dst, const uint8_t* src, int len, int lane) {
  const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + static_cast<uintptr_t>(len);
  const uintptr_t a0 = d0 & ~static_cast<uintptr_t>(15);
  const int nch = static_cast<int>((((d1 + 15) & ~static_cast<uintptr_t>(15)) - a0) >> 4);
  const uintptr_t s0 = reinterpret_cast<uintptr_t>(src);
  for (int c = lane; c < nch; c += 32) {
    const uintptr_t A = a0 + 16 * static_cast<uintptr_t>(c);
    if (A >= d0 && A + 16 <= d1) {
      stg128(A, src ? window16(s0 + (A - d0), 0, 16) : make_uint4(0, 0, 0, 0));
    } else {
      const uintptr_t lo = A > d0 ? A : d0, hi = (A + 16) < d1 ? (A + 16) : d1;
      for (uintptr_t b = lo; b < hi; ++b)
        *reinterpret_cast<uint8_t*>(b) = src ? __ldg(src + (b - d0)) : 0;
    }
  }
}

enum : int { kChunkNone = 0, kChunkZero = 1, kChunkCopy = 2, kChunkMerge = 3 };

__global__ void __launch_bounds__(kGatherThreads, TG_GATHER_MIN_BLOCKS) gather_kernel(const GatherArgs a) {
  __shared__ Job sj[kGatherMaxJobs];
  __shared__ RowIv siv[kGatherWarps][kGatherMaxJobs];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nunits = *a.units;
  const size_t canvas_bytes = static_cast<size_t>(a.M) * a.N * 3;
  const int row_len = 3 * a.M;
  const bool aligned_rows =
      (row_len & 15) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
  const int nch = row_len >> 4;  // chunks per row on the aligned path
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int k = u / a.nbands, b = u - k * a.nbands;
    const uint2 range = a.ranges[k];
    const int cnt = static_cast<int>(range.y);
    const Job* gj = a.jobs + range.x;
    const int b0 = b * kGatherBand, b1 = min(a.N, b0 + kGatherBand);
    uint8_t* canvas = a.out + static_cast<size_t>(k) * canvas_bytes;
    const uintptr_t cbase = reinterpret_cast<uintptr_t>(canvas);

    if (!(aligned_rows && cnt <= kGatherMaxJobs)) {
      // ---- fallback: rect by rect ----
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
      continue;
    }

    __syncthreads();
    for (int i = tid; i < cnt; i += kGatherThreads) sj[i] = gj[i];
    __syncthreads();
    RowIv* iv = siv[warp];
    // rows b0 + warp, b0 + warp + 8, ... (interleaved: balanced across warps)
    int r = b0 + warp;
    while (r < b1) {
      // -- interval list of row r and the first row where it changes --
      int n_iv = 0, next = b1;
      for (int jb = 0; jb < cnt; jb += 32) {
        const int j = jb + lane;
        bool act = false;
        int change = 1 << 30;
        Job J{};
        if (j < cnt) {
          J = sj[j];
          const int top = J.dy + J.h;
          act = r >= J.dy && r < top;
          change = act ? top : (J.dy > r ? static_cast<int>(J.dy) : (1 << 30));
        }
        next = min(next, __reduce_min_sync(0xffffffffu, change));
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act) {
          RowIv e;
          e.s = 3 * J.dx;
          e.e = 3 * (J.dx + J.w);
          e.zero = J.src_frame < 0;
          e.pad = 0;
          e.base = e.zero ? 0
                          : reinterpret_cast<uintptr_t>(a.frames[J.src_frame]) +
                                static_cast<uintptr_t>(3 * J.sx) - static_cast<uintptr_t>(e.s) -
                                static_cast<uintptr_t>(J.dy - J.sy) * static_cast<uintptr_t>(a.pitch);
          iv[n_iv + __popc(m & ((1u << lane) - 1u))] = e;
        }
        n_iv += __popc(m);
      }
      __syncwarp();
      const int r_end = max(r + 1, min(next, b1));  // this warp's rows in [r, r_end) share the list
      // -- per segment of the row: plan this lane's chunks, stream the rows --
      for (int seg0 = 0; seg0 < nch; seg0 += kSegChunks) {
        // plan word per chunk: kind | shift << 2 | interval << 8
        uint32_t plan[kPlanChunks];
        uintptr_t q[kPlanChunks];
        int kc = 0;  // interval cursor (chunks are increasing in v)
#pragma unroll
        for (int v = 0; v < kPlanChunks; ++v) {
          const int ch = seg0 + lane + 32 * v;
          plan[v] = kChunkNone;
          q[v] = 0;
          if (ch >= nch || n_iv == 0) continue;
          const int A = 16 * ch;
          while (kc + 1 < n_iv && iv[kc + 1].s <= A) ++kc;
          const RowIv I = iv[kc];
          if (I.e >= A + 16) {
            const uintptr_t p = I.base + static_cast<uintptr_t>(A);
            q[v] = p & ~static_cast<uintptr_t>(15);
            plan[v] = (I.zero ? kChunkZero : kChunkCopy) | static_cast<uint32_t>(p & 15) << 2;
          } else {
            plan[v] = kChunkMerge | static_cast<uint32_t>(kc) << 8;
          }
        }
        for (int rr = r; rr < r_end; rr += kGatherWarps) {
          const uintptr_t roff = static_cast<uintptr_t>(rr) * static_cast<uintptr_t>(a.pitch);
          const uintptr_t drow = cbase + static_cast<uintptr_t>(rr) * row_len;
          uint4 out[kPlanChunks], hi[kPlanChunks];
#pragma unroll
          for (int v = 0; v < kPlanChunks; ++v) {  // all raw loads first (predicated)
            const bool copy = (plan[v] & 3) == kChunkCopy;
            const bool two = copy && (plan[v] & (15u << 2)) != 0;
            const uintptr_t p = q[v] + roff;
            out[v] = copy ? ldg128(p) : make_uint4(0, 0, 0, 0);
            hi[v] = two ? ldg128(p + 16) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int v = 0; v < kPlanChunks; ++v) {
            const uint32_t kind = plan[v] & 3;
            if (kind == kChunkNone) continue;
            const int sh = static_cast<int>(plan[v] >> 2 & 15);
            if (kind == kChunkCopy && sh) out[v] = realign(out[v], hi[v], sh);
            const int A = 16 * (seg0 + lane + 32 * v);
            if (kind == kChunkMerge) {
              for (int k2 = static_cast<int>(plan[v] >> 8); k2 < n_iv && iv[k2].s < A + 16; ++k2) {
                const RowIv I = iv[k2];
                if (I.zero) continue;
                const int blo = max(A, I.s) - A, bhi = min(A + 16, I.e) - A;
                merge16(out[v], window16(I.base + roff + static_cast<uintptr_t>(A), blo, bhi),
                        blo, bhi);
              }
            }
            stg128(drow + static_cast<uintptr_t>(A), out[v]);
          }
        }
      }
      __syncwarp();
      r += ((r_end - r + kGatherWarps - 1) / kGatherWarps) * kGatherWarps;  // first row >= r_end
    }
  }
}

cudaError_t launch_gather(const GatherArgs& a, int sms, cudaStream_t stream) {
  gather_kernel<<<sms * 4, kGatherThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

int gather_bands(int N) { return ceil_div(N, kGatherBand); }

}  // namespace tg
