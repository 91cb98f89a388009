// k_band.cu -- K1 band kernel: frame differencing + threshold + dilation +
// patch-grid occupancy in ONE pass over the frames (
// frozen spec DESIGN.md §3).  Nothing per-pixel leaves the SM: the raw
// foreground bitmap that K1 (k_mask.cu) writes for K1b to re-read -- 1/24 of
// the frame bytes each way -- stays in shared memory.
//
// The reference has no pixel stage (RoIs are inputs, trace.hpp:39-45); this
// kernel produces what the planner turns into them.
//
// Decomposition.  A CTA owns one band of 16 frame rows (one patch-grid cell
// row) and walks it down the frame chain, one column part (<= 60 32-pixel
// words) at a time; the CTAs of a group cover every band of the frame, so a
// group streams the same (part, frame run) slab in lock step.
//  * Row warps: warp r owns row r of the band and streams it itself -- lane 0
//    issues one cp.async.bulk per frame row (the part plus a 32-byte halo on
//    each side) into the warp's 2-slot ring, two stages ahead; a lane turns
//    two 96-byte pixel words into two raw foreground words (VABSDIFF4 + SWAR
//    compare, pixel.cuh) against the previous frame's row held in registers,
//    so each frame byte is read from HBM once.  Lane 31 computes the halo
//    words (the r pixels either side of the part).
//  * The raw rows of a frame go to a shared-memory window; the last row warp
//    to finish a frame handles it: it publishes the band's r top and r bottom
//    raw rows to a small L2-resident edge buffer (release flag per CTA), and
//    dilates the frame L earlier -- by then the neighbouring bands (other
//    CTAs of the group, co-resident under a cooperative launch) have
//    published theirs (acquire) -- vertical OR over 2r+1 rows, funnel shifts
//    with the neighbour words, popcounts and bbox masks -> packed cell
//    summaries and activity bits.
// Roofline: HBM; per frame the W*H*3 frame bytes (+64 B of halo per row and
// part boundary, 0.6 % at 4K) in, W*H/64 bytes of cells out.
#include <algorithm>

#include "kernels.cuh"
#include "pixel.cuh"

namespace tg {

constexpr int kBandRows = kCell;                 // rows per band: one cell row
constexpr int kBandPartWords = 60;               // 32-pixel words per part (2 per lane, lanes 0..29)
constexpr int kBandHalo = 32;                    // bytes staged either side of a part
constexpr int kBandSlotBytes = kBandHalo + 96 * kBandPartWords + kBandHalo;  // 5824
constexpr int kBandSlots = 2;                    // ring slots per row warp
constexpr int kBandRaw = 4;                      // frames of raw rows in shared memory (D)
constexpr int kBandLag = 2;                      // frame q is dilated when frame q+L completes
constexpr int kBandEdgeSlots = 8;                // edge-row slots per CTA in global (>= 2L + 2)
constexpr int kBandRowWords = 64;                // raw row stride (62 used: 60 words + 2 halos)
constexpr int kBandThreads = kBandRows * 32;     // 16 row warps
static_assert(kBandRaw > kBandLag + 1, "raw window must outlive the dilation lag");
static_assert(kBandEdgeSlots >= 2 * kBandLag + 2, "edge slots reused too early");

struct BandArgs {
  const uint8_t* const* cur;
  const uint8_t* const* prev;
  int n_frames, W, H, pitch, rowbytes, threshold;
  int nwords, nparts, pw;         // words per row, column parts, words per part
  int nbands, groups;             // CTA = group * nbands + band
  int kf, nslabs;                 // frames per run; slabs = parts x runs (part fastest)
  int cells_x, cells_y, act_words;
  uint32_t* cells;
  uint32_t* active;               // zeroed before the launch
  uint32_t* mask_out;             // optional dilated mask [F][H][nwords]
  uint32_t* edges;                // [grid][kBandEdgeSlots][2][R][64]
  uint32_t* flags;                // [grid] frames published (zeroed before the launch)
};

// Stage sequence of a CTA: its slabs in order, each a frame chain over the
// slab's run (prev[f0], cur[f0], cur[f0+1], ...; an extra prev stage where
// prev[f] != cur[f-1]).
struct BandCursor {
  int s, f, fend;
  bool need_prev, valid;
  __device__ __forceinline__ void open(const BandArgs& a) {
    for (; s < a.nslabs; s += a.groups) {
      f = (s / a.nparts) * a.kf;
      fend = min(a.n_frames, f + a.kf);
      if (f < fend) {
        need_prev = true;
        valid = true;
        return;
      }
    }
    valid = false;
  }
  __device__ __forceinline__ void init(const BandArgs& a, int group) {
    s = group;
    open(a);
  }
  // false when done; else *src = frame of the stage, *out = frame whose diff
  // it completes (-1: a chain start), *part = column part
  __device__ __forceinline__ bool next(const BandArgs& a, const uint8_t** src, int* out, int* part) {
    if (valid && f >= fend && !need_prev) {
      s += a.groups;
      open(a);
    }
    if (!valid) return false;
    *part = s % a.nparts;
    if (need_prev) {
      need_prev = false;
      *out = -1;
      *src = a.prev[f];
      return true;
    }
    const uint8_t* p = a.cur[f];
    *out = f++;
    need_prev = f < fend && a.prev[f] != p;
    *src = p;
    return true;
  }
};

__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int R>
struct BandShared {
  static constexpr int kWinRows = kBandRows + 2 * R;  // raw rows -R .. 15+R
  static constexpr size_t kRawBytes = size_t(kBandRaw) * kWinRows * kBandRowWords * 4;
  static constexpr size_t kRingBytes = size_t(kBandRows) * kBandSlots * kBandSlotBytes;
  static constexpr size_t kBarOff = kRawBytes + kRingBytes + 128;  // 128: halo-lane read slack
  static constexpr size_t kBytes = kBarOff + 8 * (kBandRows * kBandSlots + kBandRaw) +
                                   8 * kBandRaw + 4 * kBandRaw;
};

// Dilation of frame x (slot d of the raw window) into cells / activity bits
// (/ mask): whole warp.  Waits for the neighbouring bands' edge rows of x.
template <int R>
__device__ __forceinline__ void band_dilate(const BandArgs& a, int x, uint32_t* win, int2 m,
                                            int band, int cta, int lane) {
  constexpr int kWin = BandShared<R>::kWinRows;
  const int f = m.x, part = m.y;
  if (R > 0) {
    const int es = x % kBandEdgeSlots;
    if (lane == 0 && band > 0)
      while (ld_acquire(&a.flags[cta - 1]) < static_cast<uint32_t>(x + 1)) __nanosleep(32);
    if (lane == 1 && band < a.nbands - 1)
      while (ld_acquire(&a.flags[cta + 1]) < static_cast<uint32_t>(x + 1)) __nanosleep(32);
    __syncwarp();
    __threadfence();
    const uint2* up = reinterpret_cast<const uint2*>(
        a.edges + ((static_cast<size_t>(max(cta - 1, 0)) * kBandEdgeSlots + es) * 2 + 1) * R *
                      kBandRowWords);
    const uint2* dn = reinterpret_cast<const uint2*>(
        a.edges + (static_cast<size_t>(cta + 1) * kBandEdgeSlots + es) * 2 * R * kBandRowWords);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint2 u = band > 0 ? __ldcg(up + i * (kBandRowWords / 2) + lane) : make_uint2(0, 0);
      const uint2 v =
          band < a.nbands - 1 ? __ldcg(dn + i * (kBandRowWords / 2) + lane) : make_uint2(0, 0);
      reinterpret_cast<uint2*>(win + i * kBandRowWords)[lane] = u;
      reinterpret_cast<uint2*>(win + (R + kBandRows + i) * kBandRowWords)[lane] = v;
    }
    __syncwarp();
  }
  const int y0 = band * kBandRows;
  const int nrow = min(kBandRows, a.H - y0);
  const int wbase = part * a.pw;
  const int j0 = wbase + 2 * lane, j1 = j0 + 1;  // frame words of lanes 0..29
  const bool v0 = 2 * lane < a.pw && j0 < a.nwords;
  const bool v1 = 2 * lane + 1 < a.pw && j1 < a.nwords;
  const uint32_t lastmask = (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;
  const uint32_t keep0 = v0 ? (j0 == a.nwords - 1 ? lastmask : 0xffffffffu) : 0u;
  const uint32_t keep1 = v1 ? (j1 == a.nwords - 1 ? lastmask : 0xffffffffu) : 0u;
  const uint2* wrow = reinterpret_cast<const uint2*>(win) + lane;
  constexpr int kStride = kBandRowWords / 2;
  uint32_t any = 0;
#pragma unroll
  for (int i = 0; i < kWin; ++i) {
    const uint2 v = wrow[i * kStride];
    any |= v.x | v.y;
  }
  const int cx0 = 2 * j0;  // first of the lane's 4 cells
  const size_t cbase = (static_cast<size_t>(f) * a.cells_y + band) * a.cells_x;
  uint32_t* mrow = a.mask_out ? a.mask_out + (static_cast<size_t>(f) * a.H + y0) * a.nwords : nullptr;
  if (!__any_sync(0xffffffffu, any != 0)) {  // empty window: zero cells (and mask rows)
    if (v0) {
      a.cells[cbase + cx0] = 0u;
      if (cx0 + 1 < a.cells_x) a.cells[cbase + cx0 + 1] = 0u;
    }
    if (v1) {
      a.cells[cbase + cx0 + 2] = 0u;
      if (cx0 + 3 < a.cells_x) a.cells[cbase + cx0 + 3] = 0u;
    }
    if (mrow) {
      for (int ly = 0; ly < nrow; ++ly) {
        if (v0) mrow[static_cast<size_t>(ly) * a.nwords + j0] = 0u;
        if (v1) mrow[static_cast<size_t>(ly) * a.nwords + j1] = 0u;
      }
    }
    return;
  }
  // raw row: words 0..pw-1 of the part, the right halo at pw, the left halo at
  // 63 (lane 31's hi), so both neighbours are plain lane rotations
  const int src_l = (lane + 31) & 31, src_r = (lane + 1) & 31;
  int occ0 = 0, occ1 = 0, occ2 = 0, occ3 = 0;
  uint32_t cols0 = 0, cols1 = 0, rows0 = 0, rows1 = 0, rows2 = 0, rows3 = 0;
  uint2 wv[2 * R + 1];
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) wv[i] = wrow[i * kStride];
#pragma unroll
  for (int ly = 0; ly < kBandRows; ++ly) {
    wv[2 * R] = wrow[(ly + 2 * R) * kStride];
    uint32_t lo = wv[0].x, hi = wv[0].y;
#pragma unroll
    for (int k = 1; k <= 2 * R; ++k) {
      lo |= wv[k].x;
      hi |= wv[k].y;
    }
#pragma unroll
    for (int k = 0; k < 2 * R; ++k) wv[k] = wv[k + 1];
    const uint32_t left = __shfl_sync(0xffffffffu, hi, src_l);
    const uint32_t right = __shfl_sync(0xffffffffu, lo, src_r);
    uint32_t d0 = lo, d1 = hi;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      d0 |= __funnelshift_r(lo, hi, k) | __funnelshift_l(left, lo, k);
      d1 |= __funnelshift_r(hi, right, k) | __funnelshift_l(lo, hi, k);
    }
    const bool in = ly < nrow;
    d0 &= in ? keep0 : 0u;
    d1 &= in ? keep1 : 0u;
    if (mrow && in) {
      if (v0) mrow[static_cast<size_t>(ly) * a.nwords + j0] = d0;
      if (v1) mrow[static_cast<size_t>(ly) * a.nwords + j1] = d1;
    }
    const uint32_t h0 = d0 >> 16, h1 = d1 >> 16;
    occ0 += __popc(d0 & 0xffffu);
    occ1 += __popc(h0);
    occ2 += __popc(d1 & 0xffffu);
    occ3 += __popc(h1);
    cols0 |= d0;
    cols1 |= d1;
    rows0 |= min(d0 & 0xffffu, 1u) << ly;
    rows1 |= min(h0, 1u) << ly;
    rows2 |= min(d1 & 0xffffu, 1u) << ly;
    rows3 |= min(h1, 1u) << ly;
  }
  uint32_t bits = 0;
  if (v0) {
    a.cells[cbase + cx0] = pack_cell(occ0, cols0 & 0xffffu, rows0);
    bits |= occ0 > 0 ? 1u : 0u;
    if (cx0 + 1 < a.cells_x) {
      a.cells[cbase + cx0 + 1] = pack_cell(occ1, cols0 >> 16, rows1);
      bits |= occ1 > 0 ? 2u : 0u;
    }
  }
  if (v1) {
    a.cells[cbase + cx0 + 2] = pack_cell(occ2, cols1 & 0xffffu, rows2);
    bits |= occ2 > 0 ? 4u : 0u;
    if (cx0 + 3 < a.cells_x) {
      a.cells[cbase + cx0 + 3] = pack_cell(occ3, cols1 >> 16, rows3);
      bits |= occ3 > 0 ? 8u : 0u;
    }
  }
  if (bits) {  // cx0 is even: the lane's 4 cells span at most two activity words
    uint32_t* act = a.active + (static_cast<size_t>(f) * a.cells_y + band) * a.act_words + (cx0 >> 5);
    const int sh = cx0 & 31;
    atomicOr(act, bits << sh);
    if (sh > 28 && (bits >> (32 - sh))) atomicOr(act + 1, bits >> (32 - sh));
  }
}

template <bool kLow, int R>
__global__ void __launch_bounds__(kBandThreads, 1) mask_band_kernel(const BandArgs a) {
  using SH = BandShared<R>;
  constexpr int kWin = SH::kWinRows;
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* raw_s = reinterpret_cast<uint32_t*>(smem);  // [kBandRaw][kWin][64]
  uint8_t* ring = smem + SH::kRawBytes;                   // [16][kBandSlots][kBandSlotBytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SH::kBarOff);
  uint64_t* dilbar = full + kBandRows * kBandSlots;       // frame slot d dilated
  int2* meta = reinterpret_cast<int2*>(dilbar + kBandRaw);  // (frame, part) of slot d
  uint32_t* cnt = reinterpret_cast<uint32_t*>(meta + kBandRaw);  // row warps done with slot d
  const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x, band = cta % a.nbands, group = cta / a.nbands;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBandRows * kBandSlots; ++s) mbar_init(&full[s], 1);
    for (int d = 0; d < kBandRaw; ++d) {
      mbar_init(&dilbar[d], 1);
      cnt[d] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  // frames this CTA (and every CTA of its group) completes
  int Q = 0;
  for (int s = group; s < a.nslabs; s += a.groups) {
    const int f0 = (s / a.nparts) * a.kf;
    Q += max(0, min(a.n_frames, f0 + a.kf) - f0);
  }
  const int y0 = band * kBandRows, y = y0 + r;
  const bool live = y < a.H;
  const uint32_t t1 =
      static_cast<uint32_t>(kLow ? a.threshold + 1 : a.threshold - 127) * 0x01010101u;
  const uint32_t lastmask = (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;
  const uint32_t halo_r_mask = R > 0 ? (1u << R) - 1u : 0u;
  const uint32_t halo_l_mask = R > 0 ? ~0u << (32 - R) : 0u;

  // issue cursor (lane 0): the ring's next fill, kBandSlots stages ahead
  BandCursor ic;
  ic.init(a, group);
  int ik = 0;
  auto issue = [&]() {
    const uint8_t* src;
    int f, part;
    if (!ic.next(a, &src, &f, &part)) return;
    const int pb = part * a.pw * 96;
    const int lo = part > 0 ? pb - kBandHalo : pb;
    const int hi = part < a.nparts - 1 ? pb + a.pw * 96 + kBandHalo : a.rowbytes;
    const int slot = r * kBandSlots + ik;
    uint8_t* dst = ring + static_cast<size_t>(slot) * kBandSlotBytes + (lo - (pb - kBandHalo));
    mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(hi - lo));
    bulk_g2s(dst, src + static_cast<size_t>(y) * a.pitch + lo, static_cast<uint32_t>(hi - lo),
             &full[slot]);
    if (++ik == kBandSlots) ik = 0;
  };
  if (live && lane == 0)
    for (int k = 0; k < kBandSlots; ++k) issue();

  BandCursor cc;
  cc.init(a, group);
  uint32_t fpar = 0;
  int k = 0, q = 0;
  uint4 P0[6] = {}, P1[6] = {};
  const uint8_t* src;
  int f, part;
  while (cc.next(a, &src, &f, &part)) {
    const bool hlane = lane == 31;
    const int wbase = part * a.pw;
    const bool v0 = 2 * lane < a.pw && wbase + 2 * lane < a.nwords;
    const bool v1 = 2 * lane + 1 < a.pw && wbase + 2 * lane + 1 < a.nwords;
    const bool hr = hlane && part < a.nparts - 1, hl = hlane && part > 0;
    uint4 C0[6] = {}, C1[6] = {};
    if (live) {
      const int slot = r * kBandSlots + k;
      mbar_wait_sleep(&full[slot], (fpar >> k) & 1u);
      fpar ^= 1u << k;
      const uint8_t* sp = ring + static_cast<size_t>(slot) * kBandSlotBytes;
      // lanes: words 2l, 2l+1 of the part; lane 31: (right halo, left halo)
      if (v0 || hr) load96(C0, sp + (hlane ? kBandHalo + 96 * a.pw : kBandHalo + 192 * lane));
      if (v1 || hl) load96(C1, sp + (hlane ? kBandHalo - 96 : kBandHalo + 192 * lane + 96));
      fence_proxy_async_shared();  // the slot's reads precede its refill
      __syncwarp();
      if (lane == 0) issue();
      if (++k == kBandSlots) k = 0;
    }
    if (f < 0) {  // chain start: this row is only the next diff's `prev`
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        P0[i] = C0[i];
        P1[i] = C1[i];
      }
      continue;
    }
    uint32_t w0 = 0, w1 = 0;
    if (live) {
      w0 = fg_word<kLow>(C0, P0, t1);
      w1 = fg_word<kLow>(C1, P1, t1);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      P0[i] = C0[i];
      P1[i] = C1[i];
    }
    if (hlane) {
      w0 = hr ? (w0 & halo_r_mask) : 0u;
      w1 = hl ? (w1 & halo_l_mask) : 0u;
    } else {
      w0 = v0 ? (wbase + 2 * lane == a.nwords - 1 ? w0 & lastmask : w0) : 0u;
      w1 = v1 ? (wbase + 2 * lane + 1 == a.nwords - 1 ? w1 & lastmask : w1) : 0u;
    }
    // raw row by index: words 0..pw-1, the right halo at pw, the left halo at 63
    const uint32_t h_r = __shfl_sync(0xffffffffu, w0, 31), h_l = __shfl_sync(0xffffffffu, w1, 31);
    if (2 * lane == a.pw) w0 = h_r;
    if (2 * lane + 1 == a.pw) w1 = h_r;
    if (hlane) {
      w0 = 0u;
      w1 = h_l;
    }
    const int d = q % kBandRaw;
    if (q >= kBandRaw) mbar_wait_sleep(&dilbar[d], ((q / kBandRaw) - 1) & 1);
    uint32_t* win = raw_s + static_cast<size_t>(d) * kWin * kBandRowWords;
    reinterpret_cast<uint2*>(win + (R + r) * kBandRowWords)[lane] = make_uint2(w0, w1);
    if (r == 0 && lane == 0) meta[d] = make_int2(f, part);
    __threadfence_block();
    __syncwarp();
    uint32_t old = 0;
    if (lane == 0) old = atomicAdd(&cnt[d], 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == kBandRows - 1) {
      // ---- last row of frame q: publish its edge rows, dilate frame q - L ----
      __threadfence_block();
      if (lane == 0) cnt[d] = 0;
      // events in frame order: frame q-1's event has dilated frame q-1-L
      if (q >= kBandLag + 1) {
        const int pq = q - 1 - kBandLag;
        mbar_wait_sleep(&dilbar[pq % kBandRaw], (pq / kBandRaw) & 1);
      }
      if (R > 0) {
        uint32_t* e = a.edges + (static_cast<size_t>(cta) * kBandEdgeSlots + q % kBandEdgeSlots) * 2 *
                                    R * kBandRowWords;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          reinterpret_cast<uint2*>(e + i * kBandRowWords)[lane] =
              reinterpret_cast<const uint2*>(win + (R + i) * kBandRowWords)[lane];
          reinterpret_cast<uint2*>(e + (R + i) * kBandRowWords)[lane] =
              reinterpret_cast<const uint2*>(win + (kBandRows + i) * kBandRowWords)[lane];
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(&a.flags[cta], static_cast<uint32_t>(q + 1));
      }
      const int x_lo = q >= kBandLag ? q - kBandLag : 0;
      const int x_hi = q == Q - 1 ? Q - 1 : q - kBandLag;  // the last event drains the lag
      for (int x = x_lo; x <= x_hi; ++x) {
        const int dx = x % kBandRaw;
        uint32_t* wx = raw_s + static_cast<size_t>(dx) * kWin * kBandRowWords;
        band_dilate<R>(a, x, wx, meta[dx], band, cta, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&dilbar[dx]);
      }
    }
    ++q;
  }
}

// ---- host launcher ---------------------------------------------------------
static SmemOptIn g_band_smem[2][kMaxRadius + 1];

template <bool kLow, int R>
static cudaError_t launch_band_t(const BandArgs& a, int grid, cudaStream_t stream) {
  const int smem = static_cast<int>(BandShared<R>::kBytes);
  cudaError_t e = g_band_smem[kLow][R].ensure(mask_band_kernel<kLow, R>, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBandThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // neighbouring bands wait on each other
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mask_band_kernel<kLow, R>, a);
}

size_t band_edge_words(int radius, int sms) {
  return static_cast<size_t>(sms) * kBandEdgeSlots * 2 * std::max(radius, 1) * kBandRowWords;
}

bool band_supported(int W, int H, int sms) {
  return ceil_div(H, kBandRows) <= sms && W >= 16;
}

cudaError_t launch_mask_band(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                             int n_frames, int W, int H, int pitch, int threshold, int radius,
                             uint32_t* d_cells, uint32_t* d_active, uint32_t* d_mask,
                             uint32_t* d_flags, size_t flag_words, uint32_t* d_edges, int sms,
                             cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  if (radius < 0 || radius > kMaxRadius) return cudaErrorInvalidValue;
  if (!band_supported(W, H, sms)) return cudaErrorNotSupported;
  BandArgs a{};
  a.cur = d_cur;
  a.prev = d_prev;
  a.n_frames = n_frames;
  a.W = W;
  a.H = H;
  a.pitch = pitch;
  a.rowbytes = 3 * W;
  a.threshold = threshold;
  a.nwords = ceil_div(W, 32);
  a.nparts = ceil_div(a.nwords, kBandPartWords);
  a.pw = ceil_div(a.nwords, a.nparts);
  a.nbands = ceil_div(H, kBandRows);
  // groups of CTAs covering the frame; each group takes every groups-th slab
  int groups = std::max(1, sms / a.nbands);
  a.kf = ceil_div(n_frames, groups);
  const int nruns = ceil_div(n_frames, a.kf);
  a.nslabs = a.nparts * nruns;
  a.groups = std::min(groups, a.nslabs);
  a.cells_x = ceil_div(W, kCell);
  a.cells_y = a.nbands;
  a.act_words = ceil_div(a.cells_x, 32);
  a.cells = d_cells;
  a.active = d_active;
  a.mask_out = d_mask;
  a.edges = d_edges;
  a.flags = d_flags;
  const int grid = a.groups * a.nbands;
  if (static_cast<size_t>(grid) > flag_words) return cudaErrorInvalidConfiguration;
  const size_t act = static_cast<size_t>(n_frames) * a.cells_y * a.act_words;
  cudaError_t e;
  if (d_active == d_flags + flag_words) {  // one allocation: one memset clears both
    e = cudaMemsetAsync(d_flags, 0, sizeof(uint32_t) * (flag_words + act), stream);
  } else {
    e = cudaMemsetAsync(d_flags, 0, sizeof(uint32_t) * grid, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_active, 0, sizeof(uint32_t) * act, stream);
  }
  if (e != cudaSuccess) return e;
  const bool low = threshold <= 127;
  switch (radius) {
#define TG_BAND_CASE(R)                                                                   \
  case R:                                                                                 \
    e = low ? launch_band_t<true, R>(a, grid, stream) : launch_band_t<false, R>(a, grid, stream); \
    break;
    TG_BAND_CASE(0) TG_BAND_CASE(1) TG_BAND_CASE(2) TG_BAND_CASE(3) TG_BAND_CASE(4)
    TG_BAND_CASE(5) TG_BAND_CASE(6) TG_BAND_CASE(7) TG_BAND_CASE(8)
#undef TG_BAND_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tg
