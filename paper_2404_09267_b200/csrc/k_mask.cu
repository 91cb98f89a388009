// k_mask.cu -- K1: fused frame differencing + threshold + dilation +
// patch-grid occupancy (frozen spec DESIGN.md §3).
//
// The reference has no pixel stage (RoIs are inputs, trace.hpp:39-45); this
// kernel produces them.  One persistent CTA per SM streams work items
// (frame, 128-row segment) in frame-fastest order, so frame t's rows are
// read as `cur` by item (t, s) and as `prev` by item (t+1, s) at about the
// same time and the second read is served from L2.
//
// Per item the rows [s0-r, s1+r) of cur and prev stream through a 4-stage
// ring of shared-memory slots filled by cp.async.bulk (TMA bulk engine,
// mbarrier completion).  Each thread turns 96 bytes (32 RGB pixels) into
// one 32-bit raw-foreground word with packed SIMD byte ops, words go to a
// 32-row smem ring, and once r rows of look-ahead exist each output row is
// dilated (vertical OR over 2r+1 ring rows, horizontal funnel-shift OR) and
// folded into per-cell occupancy (popc) and bbox bit-masks held in
// registers.  A finished cell row is written as packed u32 summaries plus a
// ballot-built activity bitmask.  HBM traffic is the frames themselves; the
// outputs are ~0.5% of it.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace tg {

constexpr int kK1Threads = 256;
constexpr int kK1Ring = 32;            // fg0 rows held (>= 2*rows_per_stage + 2*radius)
constexpr int kK1MaxWords = kK1Threads; // one output word per thread: width <= 8192
constexpr int kK1SegRows = 128;        // rows per work item (multiple of kCell)
constexpr int kK1StageTarget = 48 * 1024;

struct MaskArgs {
  const uint8_t* const* cur;
  const uint8_t* const* prev;
  int n_frames, W, H, pitch, rowbytes, threshold, radius;
  int nwords;          // ceil(W/32)
  int cells_x, cells_y, act_words;
  int rows_per_stage;  // RP
  int nstages;         // smem slots
  int nseg, total_items;
  uint32_t* cells;     // [F][cells_y][cells_x]
  uint32_t* active;    // [F][cells_y][act_words]
  uint32_t* mask_out;  // optional [F][H][nwords]
};

struct ItemCursor {
  int item, st, nst, f, s0, s1, ya, yb;
};

__device__ __forceinline__ void cursor_load(ItemCursor& c, const MaskArgs& a) {
  if (c.item >= a.total_items) return;
  c.f = c.item % a.n_frames;
  const int seg = c.item / a.n_frames;
  c.s0 = seg * kK1SegRows;
  c.s1 = min(a.H, c.s0 + kK1SegRows);
  c.ya = max(0, c.s0 - a.radius);
  c.yb = min(a.H, c.s1 + a.radius);
  c.nst = ceil_div(c.yb - c.ya, a.rows_per_stage);
  c.st = 0;
}

__device__ __forceinline__ void cursor_next(ItemCursor& c, const MaskArgs& a) {
  if (++c.st >= c.nst) {
    c.item += gridDim.x;
    cursor_load(c, a);
  }
}

// Per-byte "d > T" flag in bit 7 of each byte, SWAR without cross-byte
// borrows.  kLow (T <= 127): t1 = (T+1)*0x01010101; otherwise t1 =
// (T-127)*0x01010101 and only bytes with their top bit set can pass.
template <bool kLow>
__device__ __forceinline__ uint32_t gt_bytes(uint32_t d, uint32_t t1) {
  if (kLow) return d | ((d | 0x80808080u) - t1);
  return d & (((d & 0x7f7f7f7fu) | 0x80808080u) - t1);
}

// 4 pixels (12 bytes) of cur/prev -> 4 foreground bits (max_c |cur-prev| > T
// <=> some channel's |cur-prev| > T).
template <bool kLow>
__device__ __forceinline__ uint32_t fg4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t b0,
                                        uint32_t b1, uint32_t b2, uint32_t t1) {
  const uint32_t g0 = gt_bytes<kLow>(__vabsdiffu4(a0, b0), t1);
  const uint32_t g1 = gt_bytes<kLow>(__vabsdiffu4(a1, b1), t1);
  const uint32_t g2 = gt_bytes<kLow>(__vabsdiffu4(a2, b2), t1);
  // Planar regroup: R=[p0.c0 p1.c0 p2.c0 p3.c0], G=[..c1], B=[..c2].
  const uint32_t r = __byte_perm(__byte_perm(g0, g1, 0x0630), g2, 0x5210);
  const uint32_t g = __byte_perm(__byte_perm(g0, g1, 0x0741), g2, 0x6210);
  const uint32_t b = __byte_perm(__byte_perm(g0, g1, 0x0052), g2, 0x7410);
  // bits 7/15/23/31 -> bits 28..31 with one multiply (no colliding terms).
  return (((r | g | b) & 0x80808080u) * 0x00204081u) >> 28;
}

// 32 pixels (96 bytes, or 48 for a trailing half word) -> 32 raw fg bits.
template <bool kLow>
__device__ __forceinline__ uint32_t fg_word(const uint8_t* cs, const uint8_t* ps, int nbytes,
                                            uint32_t t4) {
  uint32_t bits = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbytes <= 48) break;
    const uint4 c0 = lds128(cs + 48 * h), c1 = lds128(cs + 48 * h + 16), c2 = lds128(cs + 48 * h + 32);
    const uint4 p0 = lds128(ps + 48 * h), p1 = lds128(ps + 48 * h + 16), p2 = lds128(ps + 48 * h + 32);
    uint32_t v = 0;
    v |= fg4<kLow>(c0.x, c0.y, c0.z, p0.x, p0.y, p0.z, t4);
    v |= fg4<kLow>(c0.w, c1.x, c1.y, p0.w, p1.x, p1.y, t4) << 4;
    v |= fg4<kLow>(c1.z, c1.w, c2.x, p1.z, p1.w, p2.x, t4) << 8;
    v |= fg4<kLow>(c2.y, c2.z, c2.w, p2.y, p2.z, p2.w, t4) << 12;
    bits |= v << (16 * h);
  }
  return bits;
}

__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

__device__ __forceinline__ uint32_t pack_cell(int occ, uint32_t cols, uint32_t rows) {
  if (occ == 0) return 0u;
  const uint32_t x0 = __ffs(cols) - 1, x1 = 31 - __clz(cols);
  const uint32_t y0 = __ffs(rows) - 1, y1 = 31 - __clz(rows);
  return static_cast<uint32_t>(occ) | x0 << 9 | x1 << 13 | y0 << 17 | y1 << 21;
}

__global__ void __launch_bounds__(kK1Threads, 1) mask_cells_kernel(const MaskArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int NS = a.nstages, RP = a.rows_per_stage;
  const int slot_bytes = 2 * RP * a.rowbytes;
  uint8_t* slots = smem;
  uint32_t* ring = reinterpret_cast<uint32_t*>(smem + NS * slot_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kK1Ring * kK1MaxWords);
  const int tid = threadIdx.x;
  const bool t_low = a.threshold <= 127;
  const uint32_t t1 = static_cast<uint32_t>(t_low ? a.threshold + 1 : a.threshold - 127) * 0x01010101u;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // Producer cursor (thread 0 only) runs NS stages ahead of the consumers.
  ItemCursor pc{static_cast<int>(blockIdx.x), 0, 0, 0, 0, 0, 0, 0};
  cursor_load(pc, a);
  auto issue = [&](long long g) {
    const int slot = static_cast<int>(g % NS);
    const int y0 = pc.ya + pc.st * RP;
    const int nr = min(RP, pc.yb - y0);
    const uint32_t bytes = static_cast<uint32_t>(nr * a.rowbytes);
    uint8_t* dc = slots + slot * slot_bytes;
    uint8_t* dp = dc + RP * a.rowbytes;
    const uint8_t* sc = a.cur[pc.f] + static_cast<size_t>(y0) * a.pitch;
    const uint8_t* sp = a.prev[pc.f] + static_cast<size_t>(y0) * a.pitch;
    mbar_arrive_expect_tx(&bars[slot], 2 * bytes);
    if (a.pitch == a.rowbytes) {
      bulk_g2s(dc, sc, bytes, &bars[slot]);
      bulk_g2s(dp, sp, bytes, &bars[slot]);
    } else {
      for (int k = 0; k < nr; ++k) {
        bulk_g2s(dc + k * a.rowbytes, sc + static_cast<size_t>(k) * a.pitch, a.rowbytes, &bars[slot]);
        bulk_g2s(dp + k * a.rowbytes, sp + static_cast<size_t>(k) * a.pitch, a.rowbytes, &bars[slot]);
      }
    }
    cursor_next(pc, a);
  };
  long long issued = 0;
  if (tid == 0) {
    while (issued < NS && pc.item < a.total_items) issue(issued++);
  }

  // Consumer state (identical in every thread).
  ItemCursor cc{static_cast<int>(blockIdx.x), 0, 0, 0, 0, 0, 0, 0};
  cursor_load(cc, a);
  long long g = 0;          // stage counter
  long long ring_base = 0;  // ring row of this item's row ya
  long long ring_next = 0;  // ring row counter
  int out_next = 0;         // next output row of the current item
  const int w = tid;        // output word owned in the dilation phase
  const bool owns_word = w < a.nwords;
  const bool in_warp_range = w < ((a.nwords + 31) & ~31);
  int occ_lo = 0, occ_hi = 0;
  uint32_t col_lo = 0, col_hi = 0, row_lo = 0, row_hi = 0;
  const uint32_t lastmask =
      (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;

  while (cc.item < a.total_items) {
    if (cc.st == 0) {
      ring_base = ring_next;
      out_next = cc.s0;
    }
    const int slot = static_cast<int>(g % NS);
    const uint32_t parity = static_cast<uint32_t>((g / NS) & 1);
    const int y0 = cc.ya + cc.st * RP;
    const int nr = min(RP, cc.yb - y0);
    mbar_wait(&bars[slot], parity);

    // ---- raw foreground words for the nr rows of this stage ----
    const uint8_t* sc = slots + slot * slot_bytes;
    const uint8_t* sp = sc + RP * a.rowbytes;
    for (int it = tid; it < nr * a.nwords; it += kK1Threads) {
      const int k = it / a.nwords, ww = it - k * a.nwords;
      const int off = 96 * ww;
      const int nbytes = min(96, a.rowbytes - off);
      const uint8_t* cw = sc + k * a.rowbytes + off;
      const uint8_t* pw = sp + k * a.rowbytes + off;
      uint32_t f = t_low ? fg_word<true>(cw, pw, nbytes, t1) : fg_word<false>(cw, pw, nbytes, t1);
      if (ww == a.nwords - 1) f &= lastmask;
      const long long rr = ring_base + (y0 - cc.ya) + k;
      ring[(rr & (kK1Ring - 1)) * kK1MaxWords + ww] = f;
    }
    ring_next = ring_base + (y0 - cc.ya) + nr;
    __syncthreads();
    if (tid == 0 && pc.item < a.total_items) {
      fence_proxy_async_smem();
      issue(g + NS);
    }

    // ---- dilation + cell accumulation for rows that now have look-ahead ----
    const int y_last = y0 + nr - 1;
    const bool item_done = (cc.st == cc.nst - 1);
    const int out_hi = item_done ? cc.s1 - 1 : min(cc.s1 - 1, y_last - a.radius);
    if (in_warp_range) {
      for (int y = out_next; y <= out_hi; ++y) {
        uint32_t vm = 0, vc = 0, vp = 0;
        const int lo = max(y - a.radius, 0), hi = min(y + a.radius, a.H - 1);
        if (owns_word) {
          for (int yy = lo; yy <= hi; ++yy) {
            const uint32_t* rrow = ring + ((ring_base + (yy - cc.ya)) & (kK1Ring - 1)) * kK1MaxWords;
            vc |= rrow[w];
            if (w > 0) vm |= rrow[w - 1];
            if (w + 1 < a.nwords) vp |= rrow[w + 1];
          }
        }
        uint32_t d = vc;
        for (int k = 1; k <= a.radius; ++k)
          d |= __funnelshift_r(vc, vp, k) | __funnelshift_l(vm, vc, k);
        if (w == a.nwords - 1) d &= lastmask;
        if (!owns_word) d = 0;
        if (a.mask_out && owns_word)
          a.mask_out[(static_cast<size_t>(cc.f) * a.H + y) * a.nwords + w] = d;
        const uint32_t dl = d & 0xffffu, dh = d >> 16;
        const int ly = y & (kCell - 1);
        occ_lo += __popc(dl);
        occ_hi += __popc(dh);
        col_lo |= dl;
        col_hi |= dh;
        row_lo |= (dl ? 1u : 0u) << ly;
        row_hi |= (dh ? 1u : 0u) << ly;
        if (ly == kCell - 1 || y == a.H - 1) {
          const int cy = y / kCell;
          const size_t cbase = (static_cast<size_t>(cc.f) * a.cells_y + cy) * a.cells_x;
          if (owns_word) {
            const int cx = 2 * w;
            a.cells[cbase + cx] = pack_cell(occ_lo, col_lo, row_lo);
            if (cx + 1 < a.cells_x) a.cells[cbase + cx + 1] = pack_cell(occ_hi, col_hi, row_hi);
          }
          const uint32_t blo = __ballot_sync(0xffffffffu, occ_lo > 0);
          const uint32_t bhi = __ballot_sync(0xffffffffu, occ_hi > 0);
          const int lane = tid & 31, wq = tid >> 5;
          const size_t abase = (static_cast<size_t>(cc.f) * a.cells_y + cy) * a.act_words;
          if (lane < 2 && 2 * wq + lane < a.act_words) {
            const uint32_t lo16 = lane ? (blo >> 16) : blo, hi16 = lane ? (bhi >> 16) : bhi;
            a.active[abase + 2 * wq + lane] = spread16(lo16) | (spread16(hi16) << 1);
          }
          occ_lo = occ_hi = 0;
          col_lo = col_hi = row_lo = row_hi = 0;
        }
      }
    }
    out_next = max(out_next, out_hi + 1);  // stages of pure look-behind halo output nothing
    ++g;
    cursor_next(cc, a);
  }
}

// ---- host launcher ---------------------------------------------------------
struct MaskPlan {
  int rows_per_stage, nstages;
  size_t smem;
};

MaskPlan plan_mask(int W) {
  const int rowbytes = 3 * W;
  MaskPlan p;
  p.rows_per_stage = std::max(1, std::min(8, kK1StageTarget / (2 * rowbytes)));
  const size_t fixed = static_cast<size_t>(kK1Ring) * kK1MaxWords * 4 + 8 * 8;
  p.nstages = 4;
  while (p.nstages > 2 &&
         fixed + static_cast<size_t>(p.nstages) * 2 * p.rows_per_stage * rowbytes > 227 * 1024)
    --p.nstages;
  p.smem = fixed + static_cast<size_t>(p.nstages) * 2 * p.rows_per_stage * rowbytes;
  return p;
}

cudaError_t launch_mask_cells(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                              int n_frames, int W, int H, int pitch, int threshold, int radius,
                              uint32_t* d_cells, uint32_t* d_active, uint32_t* d_mask, int sms,
                              cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  MaskArgs a;
  a.cur = d_cur;
  a.prev = d_prev;
  a.n_frames = n_frames;
  a.W = W;
  a.H = H;
  a.pitch = pitch;
  a.rowbytes = 3 * W;
  a.threshold = threshold;
  a.radius = radius;
  a.nwords = ceil_div(W, 32);
  a.cells_x = ceil_div(W, kCell);
  a.cells_y = ceil_div(H, kCell);
  a.act_words = ceil_div(a.cells_x, 32);
  const MaskPlan mp = plan_mask(W);
  a.rows_per_stage = mp.rows_per_stage;
  a.nstages = mp.nstages;
  a.nseg = ceil_div(H, kK1SegRows);
  a.total_items = a.nseg * n_frames;
  a.cells = d_cells;
  a.active = d_active;
  a.mask_out = d_mask;
  cudaError_t e = cudaFuncSetAttribute(mask_cells_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(mp.smem));
  if (e != cudaSuccess) return e;
  int grid = std::min(a.total_items, sms);
  if (const char* g = std::getenv("TG_K1_GRID")) grid = std::max(1, std::min(a.total_items, std::atoi(g)));
  mask_cells_kernel<<<grid, kK1Threads, mp.smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace tg
