// k_gather.cu -- K5: batched canvas writer (the paper's
// invoke(canvases) input).
//
// Every canvas is exactly tiled by its placements plus its final guillotine
// free rects: each canvas row is a left-to-right
// sequence of intervals, each either a patch's source row or zeros.  A
// persistent grid claims (canvas, band of rows) units from a device counter
// -- their count is what the planner left in device memory (no host
// round trip between planning and gathering); dynamic claiming keeps CTAs
// that drew light, zero-fill bands busy, so the grid drains together (static
// round robin: 0.82 ms vs 0.66 ms per 300 4K frames); bands are 64 rows, or
// up to 512 for long explicit plans (gather_band).  Warp w of a block
// owns rows b0 + w, b0 + w + 8, ... of the band, split into 3 KB destination
// segments ("items").
//
// Each warp runs its own TMA pipeline.  Producer side (whole warp): ballot
// the jobs active in the item's row, write the interval list into a header
// slot and, per copy interval, issue ONE cp.async.bulk of the 16-byte-aligned
// source span into a per-warp byte ring in shared memory, completing on the
// slot's mbarrier.  Consumer side (the same warp, up to kSlots items later):
// wait the mbarrier, then each lane builds its 16-byte destination chunks
// from two aligned LDS.128 + funnel shifts (byte-mask merge at interval
// edges) and writes them with full STG.128.  Loads in flight are bounded by
// ring bytes, not registers, so a warp keeps several source rows in flight
// while it realigns and stores earlier ones.
//
// Fallbacks (rare, correct for any input): canvases whose rows are not
// 16-byte aligned (3*width % 16 != 0) or that hold more jobs than the smem
// job cache go rect by rect; an item with more than kMaxIv intervals or an
// unaligned frame pointer is copied directly from global memory.
#include "kernels.cuh"

namespace tg {

#ifndef TG_GATHER_SLOTS
#define TG_GATHER_SLOTS 6
#endif
// 4: the register budget of 4 CTAs per SM (64 registers, no spills) -- the
// grid stays smem-limited at 3 per SM, and a capped event gather (configs
// 3/4, 2 per SM) leaves more registers to the K1b / planner CTAs beside it
// (config-4 pass -0.5 % against 80 registers)
#ifndef TG_GATHER_MIN_BLOCKS
#define TG_GATHER_MIN_BLOCKS 4
#endif
#ifndef TG_GATHER_RING
#define TG_GATHER_RING 6144
#endif
#ifndef TG_GATHER_DYNAMIC
#define TG_GATHER_DYNAMIC 1
#endif

// explicit plans: units per SM below which bands stay at 64 rows (gather_band)
#ifndef TG_GATHER_UNITS_PER_SM
#define TG_GATHER_UNITS_PER_SM 64LL
#endif

#ifndef TG_GATHER_THREADS
#define TG_GATHER_THREADS 256
#endif

constexpr int kGatherThreads = TG_GATHER_THREADS;
constexpr int kGatherWarps = kGatherThreads / 32;
constexpr int kGatherMaxJobs = 192;              // jobs of one canvas cached in smem
constexpr int kSlots = TG_GATHER_SLOTS;          // items in flight per warp (header slots)
constexpr int kRing = TG_GATHER_RING;            // source bytes in flight per warp
constexpr int kSegBytes = 3072;                  // destination bytes per item
constexpr int kLaneChunks = kSegBytes / 16 / 32; // 16-byte chunks per lane per item
constexpr int kMaxIv = 32;                       // intervals per segment (one per lane)
constexpr uint16_t kZeroIv = 0xffff;
enum : uint32_t { kChunkNone = 0, kChunkZero = 1, kChunkCopy = 2, kChunkMerge = 3 };
static_assert(kRing >= kSegBytes + 32 * kMaxIv + 16, "ring must hold the largest item");
static_assert(kRing < 65536 - 64, "ring offsets are 16-bit");

struct IvHdr {
  uint16_t s, e;  // destination bytes [s, e) of the segment
  uint16_t a;     // ring offset (from the item's pos) of the source byte for s
  uint16_t j;     // job index, kZeroIv for zero fill
};

// Items run in (run of rows with one interval set, segment, row) order; the
// interval list of a (run, segment) travels in the slot of its first item.
struct alignas(16) WarpStage {
  uint64_t bar[kSlots];
  int4 info[kSlots];         // pos in ring, n intervals (-1: direct), row, seg | first << 16
  IvHdr iv[kSlots][kMaxIv];  // producer -> consumer, first item of a (run, segment)
  IvHdr civ[kMaxIv];         // consumer's copy for its current (run, segment)
  uint32_t mlist[kLaneChunks * 32];  // its edge chunks: A | first interval << 16
  uint8_t pad0[16];          // realign windows may start up to 15 bytes early ...
  uint8_t ring[kRing];
  uint8_t pad1[32];          // ... and end up to 32 bytes late (masked garbage)
};

constexpr size_t kGatherSmem = sizeof(Job) * kGatherMaxJobs + sizeof(WarpStage) * kGatherWarps;

__device__ __forceinline__ uint4 ldg128(uintptr_t p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// Plain (weak) global store: __stcg would emit STG.STRONG.GPU.
__device__ __forceinline__ void stg128(uintptr_t p, const uint4& v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Bytes [s, s+16) of the 32-byte pair (v0, v1); branch-free: two levels of
// word selects (11 SEL) + funnel shifts.
__device__ __forceinline__ uint4 realign(const uint4& v0, const uint4& v1, int s) {
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  const bool q2 = (s & 8) != 0, q1 = (s & 4) != 0;
  const int sh = 8 * (s & 3);
  uint32_t t[6];  // t[j] = w[j + (q & 2)]
#pragma unroll
  for (int j = 0; j < 6; ++j) t[j] = q2 ? w[j + 2] : w[j];
  uint32_t p[5];  // p[j] = w[j + q]
#pragma unroll
  for (int j = 0; j < 5; ++j) p[j] = q1 ? t[j + 1] : t[j];
  return make_uint4(__funnelshift_r(p[0], p[1], sh), __funnelshift_r(p[1], p[2], sh),
                    __funnelshift_r(p[2], p[3], sh), __funnelshift_r(p[3], p[4], sh));
}

// 16 bytes of a global window starting at p whose bytes [need_lo, need_hi)
// are readable; aligned blocks not intersecting them are never touched, so
// reads stay inside the source row.
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

// 16 bytes at ring offset aa (may be up to 15 below the item start): five
// word loads from the 4-byte-aligned address + four funnel shifts (fewer
// instructions than two aligned LDS.128 + word selects; the 4-way bank
// conflict of 16-byte-strided lanes is affordable at this byte rate).
__device__ __forceinline__ uint4 ring16(const uint8_t* ring, int aa) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + (aa & ~3));
  const int sh = 8 * (aa & 3);
  const uint32_t w0 = p[0], w1 = p[1], w2 = p[2], w3 = p[3], w4 = p[4];
  return make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh),
                    __funnelshift_r(w2, w3, sh), __funnelshift_r(w3, w4, sh));
}

// x << n with n >= 32 giving 0 (PTX shl clamps the shift amount).
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t n) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}

// out bytes [lo, hi) := v bytes [lo, hi)   (0 <= lo < hi <= 16)
__device__ __forceinline__ void merge16(uint4& out, const uint4& v, int lo, int hi) {
  uint32_t* o = &out.x;
  const uint32_t* x = &v.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t m = shl_clamp(~0u, static_cast<uint32_t>(max(8 * lo - 32 * k, 0))) &
                       ~shl_clamp(~0u, static_cast<uint32_t>(max(8 * hi - 32 * k, 0)));
    o[k] = (o[k] & ~m) | (x[k] & m);
  }
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

// Source address of destination byte x (absolute, in the canvas row) of job
// J at canvas row `row`.
__device__ __forceinline__ uintptr_t job_src(const GatherArgs& a, const Job& J, int row, int x) {
  return reinterpret_cast<uintptr_t>(a.frames[J.src_frame]) +
         static_cast<uintptr_t>(J.sy + (row - J.dy)) * static_cast<uintptr_t>(a.pitch) +
         static_cast<uintptr_t>(3 * J.sx + (x - 3 * J.dx));
}

__global__ void __launch_bounds__(kGatherThreads, TG_GATHER_MIN_BLOCKS) gather_kernel(const GatherArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Job* sj = reinterpret_cast<Job*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpStage& W = reinterpret_cast<WarpStage*>(smem + sizeof(Job) * kGatherMaxJobs)[warp];
  if (lane < kSlots) mbar_init(&W.bar[lane], 1);
  fence_mbar_init();
  __syncwarp();

  const int nunits = *a.units;
  const size_t canvas_bytes = static_cast<size_t>(a.M) * a.N * 3;
  const int row_len = 3 * a.M;
  const bool aligned_rows =
      (row_len & 15) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
  const int nseg = ceil_div(row_len, kSegBytes);
  const unsigned lt = (1u << lane) - 1u;
  int gbase = 0;  // items this warp has pushed through its slots so far

#if TG_GATHER_DYNAMIC
  // units are claimed in order from a counter: CTAs that drew light (zero
  // fill) bands take more, so the grid drains together
  __shared__ int s_unit;
  for (;;) {
    __syncthreads();  // everyone has read the previous claim
    if (tid == 0) s_unit = atomicAdd(&a.units[1], 1);
    __syncthreads();
    const int u = s_unit;
    if (u >= nunits) break;
#else
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
#endif
    const int k = u / a.nbands, b = u - k * a.nbands;
    const uint2 range = a.ranges[k];
    const int cnt = static_cast<int>(range.y);
    const Job* gj = a.jobs + range.x;
    const int b0 = b * a.band, b1 = min(a.N, b0 + a.band);
    uint8_t* canvas = a.out + static_cast<size_t>(k) * canvas_bytes;

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

    int c = 0, p = 0, head = 0, tail = 0;  // consumed / produced items; ring [tail, head) live
    uint32_t plan[kLaneChunks];             // consumer: chunk plans of its (run, segment)
    int n_merge = 0;

    // ---- consumer: build and store the destination chunks of item c ----
    auto consume = [&]() {
      const int g = gbase + c;
      const int slot = g % kSlots;
      mbar_wait(&W.bar[slot], static_cast<uint32_t>(g / kSlots) & 1u);
      const int4 inf = W.info[slot];
      const int n = inf.y, row = inf.z, seg = inf.w & 0xffff;
      const int sB0 = seg * kSegBytes, len = min(row_len, sB0 + kSegBytes) - sB0;
      uint8_t* drow = canvas + static_cast<size_t>(row) * row_len + sB0;
      if (n < 0) {  // direct from global memory
        for (int j = 0; j < cnt; ++j) {
          const Job J = sj[j];
          const int s = 3 * J.dx, e = 3 * (J.dx + J.w);
          if (row < J.dy || row >= J.dy + J.h || e <= sB0 || s >= sB0 + len) continue;
          const int cs = max(s, sB0), ce = min(e, sB0 + len);
          const uint8_t* src =
              J.src_frame >= 0 ? reinterpret_cast<const uint8_t*>(job_src(a, J, row, cs)) : nullptr;
          copy_rect_row(drow + (cs - sB0), src, ce - cs, lane);
        }
      } else {
        if (inf.w >> 16) {  // first item of a (run, segment): take its list, plan the chunks
          if (lane < n) W.civ[lane] = W.iv[slot][lane];
          __syncwarp();
          n_merge = 0;
          int kc = 0;
#pragma unroll
          for (int v = 0; v < kLaneChunks; ++v) {
            const int A = 16 * (lane + 32 * v);
            bool merge = false;
            plan[v] = kChunkNone;
            if (A < len) {
              while (kc + 1 < n && W.civ[kc + 1].s <= A) ++kc;
              plan[v] = kChunkZero;
              if (n > 0) {
                const IvHdr I = W.civ[kc];
                if (I.s <= A && I.e >= A + 16) {
                  if (I.j != kZeroIv) plan[v] = kChunkCopy | static_cast<uint32_t>(I.a + A - I.s) << 8;
                } else {
                  plan[v] = kChunkNone;  // stored by the merge pass
                  merge = true;
                }
              }
            }
            // chunks straddling interval edges go to a compact per-warp list
            int cnt_iv = 0;  // intervals overlapping the chunk, from kc on
            if (merge)
              while (kc + cnt_iv < n && W.civ[kc + cnt_iv].s < A + 16) ++cnt_iv;
            const unsigned mm = __ballot_sync(0xffffffffu, merge);
            if (merge)
              W.mlist[n_merge + __popc(mm & lt)] = static_cast<uint32_t>(A) |
                                                   static_cast<uint32_t>(kc) << 16 |
                                                   static_cast<uint32_t>(cnt_iv) << 24;
            n_merge += __popc(mm);
          }
          __syncwarp();
        }
        const uint8_t* ring = W.ring + inf.x;
        const uintptr_t dbase = reinterpret_cast<uintptr_t>(drow);
#pragma unroll
        for (int v = 0; v < kLaneChunks; ++v) {
          const uint32_t kind = plan[v] & 3;
          const uintptr_t d = dbase + 16 * (lane + 32 * v);
          if (kind == kChunkCopy)
            stg128(d, ring16(ring, static_cast<int>(plan[v] >> 8)));
          else if (kind == kChunkZero)
            stg128(d, make_uint4(0, 0, 0, 0));
        }
        for (int i = lane; i < n_merge; i += 32) {  // edge chunks: byte-masked merge
          const uint32_t e = W.mlist[i];
          const int A = static_cast<int>(e & 0xffff);
          uint4 out = make_uint4(0, 0, 0, 0);
          const int k0 = static_cast<int>(e >> 16 & 0xff), k1 = k0 + static_cast<int>(e >> 24);
          for (int k2 = k0; k2 < k1; ++k2) {
            const IvHdr I2 = W.civ[k2];
            if (I2.j == kZeroIv || I2.e <= A) continue;
            merge16(out, ring16(ring, I2.a + A - I2.s), max(A, static_cast<int>(I2.s)) - A,
                    min(A + 16, static_cast<int>(I2.e)) - A);
          }
          stg128(dbase + A, out);
        }
      }
      __syncwarp();
      ++c;
    };

    // ---- ring placement of `total` bytes for item p (consumes until it fits) ----
    auto place = [&](int total) -> int {
      if (total == 0) return head;
      int pos;
      for (;;) {
        if (c == p)
          head = tail = 0;
        else
          tail = W.info[(gbase + c) % kSlots].x;  // oldest live item
        if (head >= tail) {
          if (head + total <= kRing) { pos = head; break; }
          if (total < tail) { pos = 0; break; }
        } else if (head + total < tail) {
          pos = head;
          break;
        }
        consume();
      }
      head = pos + total;
      return pos;
    };

    // ---- producer ----
    int r = b0 + warp;
    while (r < b1) {
      // this warp's rows in [r, r_end) share one interval set
      int next = b1;
      for (int jb = 0; jb < cnt; jb += 32) {
        const int j = jb + lane;
        int change = 1 << 30;
        if (j < cnt) {
          const Job J = sj[j];
          const int top = J.dy + J.h;
          change = (r >= J.dy && r < top) ? top : (J.dy > r ? static_cast<int>(J.dy) : (1 << 30));
        }
        next = min(next, __reduce_min_sync(0xffffffffu, change));
      }
      const int r_end = max(r + 1, min(next, b1));
      for (int seg = 0; seg < nseg; ++seg) {
        const int sB0 = seg * kSegBytes, sB1 = min(row_len, sB0 + kSegBytes);
        while (p - c >= kSlots) consume();
        IvHdr* H = W.iv[(gbase + p) % kSlots];  // travels with the first item
        // interval list of the segment in x order (a canvas' jobs are sorted by dx)
        int n = 0;
        bool direct = false;
        for (int jb = 0; jb < cnt; jb += 32) {
          const int j = jb + lane;
          bool act = false;
          IvHdr h{};
          if (j < cnt) {
            const Job J = sj[j];
            const int s = 3 * J.dx, e = 3 * (J.dx + J.w);
            act = r >= J.dy && r < J.dy + J.h && e > sB0 && s < sB1;
            h.s = static_cast<uint16_t>(max(s, sB0) - sB0);
            h.e = static_cast<uint16_t>(min(e, sB1) - sB0);
            h.j = J.src_frame < 0 ? kZeroIv : static_cast<uint16_t>(j);
          }
          const unsigned m = __ballot_sync(0xffffffffu, act);
          if (n + __popc(m) > kMaxIv) {
            direct = true;
            break;
          }
          if (act) H[n + __popc(m & lt)] = h;
          n += __popc(m);
        }
        __syncwarp();
        // lane i owns interval i: its aligned source span (row-invariant
        // shift because pitch % 16 == 0) and its ring offset
        uintptr_t q0 = 0;  // aligned source address at canvas row 0 (mod 2^64)
        int nb = 0, sh = 0;
        bool bad = false;
        if (!direct && lane < n) {
          const IvHdr h = H[lane];
          if (h.j != kZeroIv) {
            const Job J = sj[h.j];
            const uintptr_t fb = reinterpret_cast<uintptr_t>(a.frames[J.src_frame]);
            bad = (fb & 15) != 0;
            const uintptr_t src0 =
                fb + static_cast<uintptr_t>(static_cast<long long>(J.sy - J.dy) * a.pitch) +
                static_cast<uintptr_t>(3 * J.sx + (sB0 + h.s - 3 * J.dx));
            sh = static_cast<int>(src0 & 15);
            q0 = src0 - static_cast<uintptr_t>(sh);
            nb = (sh + h.e - h.s + 15) & ~15;
          }
        }
        direct = direct || __any_sync(0xffffffffu, bad);
        int incl = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int off = incl - nb;
        const int total = direct ? 0 : __shfl_sync(0xffffffffu, incl, 31);
        if (!direct && lane < n) H[lane].a = static_cast<uint16_t>(off + sh);
        __syncwarp();
        for (int rr = r; rr < r_end; rr += kGatherWarps) {
          while (p - c >= kSlots) consume();
          const int slot = (gbase + p) % kSlots;
          const int pos = place(total);
          if (lane == 0) {
            W.info[slot] = make_int4(pos, direct ? -1 : n, rr, seg | (rr == r ? 1 << 16 : 0));
            mbar_arrive_expect_tx(&W.bar[slot], static_cast<uint32_t>(total));
          }
          __syncwarp();
          if (!direct && nb > 0) {
            fence_proxy_async_smem();
            bulk_g2s(W.ring + pos + off,
                     reinterpret_cast<const void*>(q0 + static_cast<uintptr_t>(rr) *
                                                            static_cast<uintptr_t>(a.pitch)),
                     static_cast<uint32_t>(nb), &W.bar[slot]);
          }
          ++p;
        }
      }
      r += ((r_end - r + kGatherWarps - 1) / kGatherWarps) * kGatherWarps;  // first row >= r_end
    }
    while (c < p) consume();
    gbase += p;
  }
#if TG_GATHER_DYNAMIC
  if (tid == 0) {  // the last CTA out leaves the counters at 0 for the next launch
    __threadfence();
    if (atomicAdd(&a.units[2], 1) == static_cast<int>(gridDim.x) - 1) {
      a.units[1] = 0;
      a.units[2] = 0;
    }
  }
#endif
}

cudaError_t launch_gather(const GatherArgs& a, int sms, int grid_ctas, cudaStream_t stream) {
  // resident CTAs per SM, per device (0 = not yet queried)
  static std::atomic<int> blocks_per_sm[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int nb = (dev >= 0 && dev < kMaxDevices) ? blocks_per_sm[dev].load(std::memory_order_relaxed) : 0;
  if (nb == 0) {
    e = cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kGatherSmem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gather_kernel, kGatherThreads,
                                                      kGatherSmem);
    if (e != cudaSuccess) return e;
    nb = nb > 0 ? nb : 1;
    if (dev >= 0 && dev < kMaxDevices) blocks_per_sm[dev].store(nb, std::memory_order_relaxed);
  }
  const int grid = grid_ctas > 0 ? std::min(grid_ctas, sms * nb) : sms * nb;
  gather_kernel<<<grid, kGatherThreads, kGatherSmem, stream>>>(a);
  return cudaGetLastError();
}

int gather_bands(int N, int band) { return ceil_div(N, band); }

// Taller bands amortise each warp's interval lists and chunk plans over more
// rows (config 4's event gather, 3,713 canvases per pass: 64 -> 256 rows,
// pass -2 %); short plans keep 64 so the dynamic claim still balances the
// grid (config 2's per-step gather: 256 rows +4 %).
int gather_band(int n_canvases, int N, int sms) {
  int band = kGatherDefaultBand;
  while (band < 8 * kGatherDefaultBand &&
         static_cast<long long>(n_canvases) * gather_bands(N, 2 * band) >= TG_GATHER_UNITS_PER_SM * sms)
    band *= 2;
  return band;
}

}  // namespace tg
