// k_mask.cu -- K1: frame differencing + threshold (raw foreground bitmap)
// and K1b: dilation + patch-grid occupancy (frozen
// spec DESIGN.md §3).
//
// The reference has no pixel stage (RoIs are inputs, trace.hpp:39-45); these
// kernels produce them.
//
// K1 (mask_fg_kernel) -- persistent, one CTA per SM, warp-specialized, HBM
// bound.  A work item is (block of rows, run of consecutive frames).  Frame t
// is `cur` of diff t and `prev` of diff t+1 (checked on the device: prev[t]
// == cur[t-1]; a break starts a new chain), so along a chain every frame row
// is staged ONCE and each HBM byte is read once.
//  * A unit is (row, part of <= 64 32-pixel words); an item's units go one
//    per consumer group.  Each group walks its unit down the frame chain.
//  * Producer warp: lane g streams group g's frame rows (prev[f0], cur[f0],
//    cur[f0+1], ...) into the group's ring of smem slots with cp.async.bulk
//    (the TMA bulk engine) on full/empty mbarriers, polling slot release
//    with non-blocking test_wait so no group's latency stalls another's.
//  * Consumer groups of 2 warps: a lane owns one 32-pixel word of the part.
//    It loads its 96 bytes of the next frame row into registers and releases
//    the slot at once (slots turn around in a load latency, not a compute
//    time), then turns (previous row, this row) into one 32-bit raw
//    foreground word with packed SIMD byte ops (VABSDIFF4 + SWAR compare +
//    PRMT planar regroup); this row stays in registers as the next `prev`.
//  * Raw words go to global memory (1 bit/pixel: 1/24 of the frame bytes).
//
// K1b (dilate_strip) -- per (frame, 64-row strip, 30-word column group) warp
// task: vertical OR over 2r+1 raw rows, horizontal funnel shifts with
// neighbour words from adjacent lanes, per-cell popcounts and bbox bit-masks
// -> packed u32 cell summaries plus an activity bitmask (and the dilated mask
// on request).
//
// Fused launch (launch_mask_fused, the pipeline's mask stage): ~9 % of the
// CTAs run only K1b tasks, on SMs of their own, trailing the stream front;
// the others stream (the same number of items each) and then join them.
// Tasks come from a queue in strip order; a task starts once every K1 item
// covering its rows has published completion (per-item counters,
// release/acquire).  Cooperative launch guarantees that all CTAs are
// co-resident, so waiting on other CTAs' items cannot deadlock.  Measured
// alternatives (300 4K frames, mask stage; 1.276 ms with every CTA
// streaming and K1b as a tail, 1.255 ms as built): 1 / 3 / 5 extra warps per
// CTA running K1b tasks beside the stream 1.29 / 1.31 / 1.46 ms and consumer
// warps taking 1/2/4/8 ready tasks between their items 1.30 / 1.33 / 1.37 /
// 1.49 ms -- K1b on the streaming SMs slows the stream more than it hides;
// L2 evict_first on the frame stream + evict_last on the raw words cut DRAM
// reads by 0.14 GB but not time; a sparse raw bitmap (only non-zero words
// written, plus per-row ballot masks) saved K1 15 us but cost K1b 60 us in
// the fused launch (round 1).  Round 2's form (TG_K1_SPARSE, kernels.cuh):
// K1 stores only the 32-byte sectors holding a foreground bit plus one flag
// word per 32 raw words per row (parts 32-word aligned, so a consumer warp's
// ballot is one flag word), K1b loads a band's flags first, then only the
// flagged words -- config-4 pass 11.43 -> 11.29 ms, config 3 8.74 -> 8.63
// ms (split launches: the raw bitmap goes through DRAM), and with
// TG_K1_SPARSE_FUSED the config-2 step 1.959 -> 1.935 ms (same boxes).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace tg {


// Fused launch: the frame lines are streamed with evict_first (bit 0) and the
// raw words stored with evict_last (bit 1), so more of the raw rows the K1b
// tasks read back are still in L2 (300 4K frames: DRAM reads 7.86 -> 7.79
// GB, config-2 step -0.4 %).  K1b tasks trailing the stream front by 8-frame
// progress blocks (a publisher warp per CTA, a stream-order task table) on
// top of this: 7.75 GB and no faster.
#ifndef TG_K1_L2HINT
#define TG_K1_L2HINT 3
#endif

constexpr int kK1MaxPartWords = 64;     // 32-pixel words per unit (one per consumer lane)
constexpr int kK1Group = 2;             // warps per consumer group
constexpr int kK1Groups = 8;            // consumer groups (units per item)
constexpr int kK1MaxSlots = 8;          // ring slots per group
#ifndef TG_K1_DILATE_WARPS
#define TG_K1_DILATE_WARPS 0
#endif
constexpr int kK1DilateWarps = TG_K1_DILATE_WARPS;  // fused launch: extra warps running K1b tasks
constexpr int kK1Threads = (kK1Groups * kK1Group + 1 + kK1DilateWarps) * 32;
constexpr int kK1bBands = 4;            // cell bands per K1b task (a 64-row strip)
constexpr int kK1SmemBudget = 227 * 1024;
constexpr int kK1GroupWords = 30;       // K1b: output words per warp (lanes 1..30)
constexpr int kK1MaxActWords = 16;      // K1b: act words per cell row (W <= 8192)

// ---- K1b: dilation + cell summaries ---------------------------------------
struct DilateArgs {
  const uint32_t* raw;
  const uint32_t* zero;  // H * nwords zero words: the rows of columns outside the frame
  const uint32_t* flags;  // split launches, sparse bitmap: [F][H][fwords] word flags
  int H, W, nwords, fwords, cells_x, cells_y, act_words;
  uint32_t* cells;
  uint32_t* active;
  uint32_t* mask_out;
};

__device__ __forceinline__ uint32_t pack_cell(int occ, uint32_t cols, uint32_t rows) {
  if (occ == 0) return 0u;
  const uint32_t x0 = __ffs(cols) - 1, x1 = 31 - __clz(cols);
  const uint32_t y0 = __ffs(rows) - 1, y1 = 31 - __clz(rows);
  return static_cast<uint32_t>(occ) | x0 << 9 | x1 << 13 | y0 << 17 | y1 << 21;
}

// One band's 16 output rows from the raw window: vertical OR over 2R+1 rows,
// horizontal OR with the neighbour lanes' words, per-cell popcounts, column
// and row masks.  kFull: all 16 rows inside the frame; kMask: also store the
// dilated mask.
template <int R, bool kFull, bool kMask>
__device__ __forceinline__ void dilate_band(const DilateArgs& a, const uint32_t (&win)[kCell + 2 * R],
                                            uint32_t keep, int nrow, uint32_t* mrow, int& occ,
                                            int& occ_hi, uint32_t& cols, uint32_t& row_lo,
                                            uint32_t& row_hi) {
#pragma unroll
  for (int ly = 0; ly < kCell; ++ly) {
    uint32_t v = win[ly];
#pragma unroll
    for (int k = 1; k <= 2 * R; ++k) v |= win[ly + k];
    const uint32_t vm = __shfl_up_sync(0xffffffffu, v, 1);
    const uint32_t vp = __shfl_down_sync(0xffffffffu, v, 1);
    uint32_t d = v;
#pragma unroll
    for (int k = 1; k <= R; ++k) d |= __funnelshift_r(v, vp, k) | __funnelshift_l(vm, v, k);
    d &= (kFull || ly < nrow) ? keep : 0u;
    if (kMask && keep && (kFull || ly < nrow)) mrow[static_cast<size_t>(ly) * a.nwords] = d;
    occ += __popc(d);
    occ_hi += __popc(d >> 16);
    cols |= d;
    if (d & 0xffffu) row_lo |= 1u << ly;
    if (d > 0xffffu) row_hi |= 1u << ly;
  }
}

// One warp: frame f, cell rows cy0 .. cy0+3, words [30*wi - 1, 30*wi + 31)
// (lanes 1..30 own a word, lanes 0/31 are the neighbours; a lane whose column
// is outside the frame reads the zero page).  kFused: raw rows were written
// by other SMs during this launch -> L2 loads (ld.cg), activity bits straight
// to global (zeroed before the launch); otherwise the CTA's act_s collects
// them.
template <int R, bool kFused, bool kMask, bool kSparse = false>
__device__ __forceinline__ void dilate_strip(const DilateArgs& a, int f, int cy0, int wi, int lane,
                                             uint32_t (*act_s)[kK1MaxActWords]) {
  const int nb = min(kK1bBands, a.cells_y - cy0);
  const uint32_t lastmask = (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;
  const int w = wi * kK1GroupWords + lane - 1;
  const bool col_ok = w >= 0 && w < a.nwords;
  const bool owns = lane >= 1 && lane <= kK1GroupWords && col_ok;
  // bits this lane keeps: its own word, minus pixels past the frame edge
  const uint32_t keep = owns ? (w == a.nwords - 1 ? lastmask : 0xffffffffu) : 0u;
  const uint32_t* fr = col_ok ? a.raw + static_cast<size_t>(f) * a.H * a.nwords + w : a.zero;
  auto ld = [](const uint32_t* q) -> uint32_t { return kFused ? __ldcg(q) : __ldg(q); };
  // sparse bitmap: a word is loaded only if its row's flag bit is set (the
  // zero page stands in for the flags of columns outside the frame)
  const uint32_t* fl = kSparse ? (col_ok ? a.flags + static_cast<size_t>(f) * a.H * a.fwords + (w >> 5)
                                         : a.zero)
                               : nullptr;
  const uint32_t wbit = 1u << (w & 31);
  // rows outside [0, H) read a clamped row and are masked to zero
  auto raw_row = [&](int yy) -> uint32_t {
    const uint32_t m = (yy >= 0 && yy < a.H) ? 0xffffffffu : 0u;
    const int yc = min(max(yy, 0), a.H - 1);
    if (kSparse && !(ld(fl + static_cast<size_t>(yc) * a.fwords) & wbit)) return 0u;
    return ld(fr + static_cast<size_t>(yc) * a.nwords) & m;
  };
  // window of raw rows yb0 - R .. yb0 + 15 + R; consecutive bands share 2R rows
  constexpr int kWin = kCell + 2 * R;
  uint32_t win[kWin];
#pragma unroll
  for (int i = 0; i < 2 * R; ++i) win[i] = raw_row(cy0 * kCell - R + i);
  const uint32_t* q = fr + static_cast<size_t>(cy0 * kCell + R) * a.nwords;
  const uint32_t* fq = kSparse ? fl + static_cast<size_t>(cy0 * kCell + R) * a.fwords : nullptr;
  for (int bi = 0; bi < nb; ++bi, q += kCell * a.nwords, fq += kSparse ? kCell * a.fwords : 0) {
    const int yb0 = (cy0 + bi) * kCell, cy = cy0 + bi;
    const bool interior = yb0 + kCell + R <= a.H;  // uniform: no row past the frame
    if (kSparse && interior) {  // all flags first, then only the flagged words
      uint32_t fb[kCell];
#pragma unroll
      for (int i = 0; i < kCell; ++i) fb[i] = ld(fq + i * a.fwords);
#pragma unroll
      for (int i = 2 * R; i < kWin; ++i)
        win[i] = (fb[i - 2 * R] & wbit) ? ld(q + (i - 2 * R) * a.nwords) : 0u;
    } else if (interior) {
#pragma unroll
      for (int i = 2 * R; i < kWin; ++i) win[i] = ld(q + (i - 2 * R) * a.nwords);
    } else {
#pragma unroll
      for (int i = 2 * R; i < kWin; ++i) win[i] = raw_row(yb0 - R + i);
    }
    const int nrow = min(kCell, a.H - yb0);
    const size_t cbase = (static_cast<size_t>(f) * a.cells_y + cy) * a.cells_x;
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < kWin; ++i) any |= win[i];
    if (!kMask && !__any_sync(0xffffffffu, any != 0)) {  // empty band tile: zero cells
      if (owns) {
        a.cells[cbase + 2 * w] = 0u;
        if (2 * w + 1 < a.cells_x) a.cells[cbase + 2 * w + 1] = 0u;
      }
#pragma unroll
      for (int i = 0; i < 2 * R; ++i) win[i] = win[kCell + i];
      continue;
    }
    int occ = 0, occ_hi = 0;
    uint32_t cols = 0, row_lo = 0, row_hi = 0;
    uint32_t* mrow = kMask ? a.mask_out + (static_cast<size_t>(f) * a.H + yb0) * a.nwords + w : nullptr;
    if (nrow == kCell)
      dilate_band<R, true, kMask>(a, win, keep, nrow, mrow, occ, occ_hi, cols, row_lo, row_hi);
    else
      dilate_band<R, false, kMask>(a, win, keep, nrow, mrow, occ, occ_hi, cols, row_lo, row_hi);
#pragma unroll
    for (int i = 0; i < 2 * R; ++i) win[i] = win[kCell + i];
    if (owns) {
      const int cx = 2 * w;
      const int occ_lo = occ - occ_hi;
      a.cells[cbase + cx] = pack_cell(occ_lo, cols & 0xffffu, row_lo);
      if (cx + 1 < a.cells_x) a.cells[cbase + cx + 1] = pack_cell(occ_hi, cols >> 16, row_hi);
      const uint32_t bits = (occ_lo > 0 ? 1u : 0u) | (occ_hi > 0 ? 2u : 0u);
      if (bits) {
        if (kFused)
          atomicOr(&a.active[(static_cast<size_t>(f) * a.cells_y + cy) * a.act_words + (cx >> 5)],
                   bits << (cx & 31));
        else
          atomicOr(&act_s[bi][cx >> 5], bits << (cx & 31));
      }
    }
  }
}

template <int R, bool kSparse>  // dilation radius, sparse raw bitmap
__global__ void __launch_bounds__(320) dilate_cells_kernel(const DilateArgs a) {  // W <= 8192: <= 9 warps
  __shared__ uint32_t act_s[kK1bBands][kK1MaxActWords];
  const int strips = ceil_div(a.cells_y, kK1bBands);
  const int f = blockIdx.x / strips, cy0 = (blockIdx.x - f * strips) * kK1bBands;
  const int nb = min(kK1bBands, a.cells_y - cy0);
  for (int i = threadIdx.x; i < kK1bBands * kK1MaxActWords; i += blockDim.x) (&act_s[0][0])[i] = 0;
  __syncthreads();
  if (a.mask_out)
    dilate_strip<R, false, true, kSparse>(a, f, cy0, threadIdx.x >> 5, threadIdx.x & 31, act_s);
  else
    dilate_strip<R, false, false, kSparse>(a, f, cy0, threadIdx.x >> 5, threadIdx.x & 31, act_s);
  __syncthreads();
  for (int i = threadIdx.x; i < nb * a.act_words; i += blockDim.x) {
    const int bi = i / a.act_words, aw = i - bi * a.act_words;
    a.active[(static_cast<size_t>(f) * a.cells_y + cy0 + bi) * a.act_words + aw] = act_s[bi][aw];
  }
}

struct MaskArgs {
  const uint8_t* const* cur;
  const uint8_t* const* prev;
  int n_frames, W, H, pitch, rowbytes, threshold;
  int nwords, part_words, nparts;
  int rows_per_item;  // units per item = rows_per_item * nparts <= kK1Groups
  int nrb;            // row blocks
  int kf, ntg;        // frames per run, runs
  int total_items;
  int dctas;          // fused launch: CTAs 0..dctas-1 run only K1b tasks (stream on the rest)
  int nslots;         // ring slots per group
  int slot_bytes;
  uint32_t* raw;      // [F][H][nwords] raw foreground bits
  uint32_t* flags;    // split launch, sparse bitmap: [F][H][fwords] word flags (else null)
  int fwords;
  // fused launch only (item_done == nullptr otherwise)
  uint32_t* item_done;  // [total_items] warps done per item (zeroed)
  uint32_t* task_next;  // K1b task queue head (zeroed)
  int radius, dgroups, strips, n_tasks;
  DilateArgs d;
};

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
// TG_FG_MAX3=0 builds the round-1 planar-regroup form (per-byte threshold,
// 6 PRMT + 2 LOP3 to OR each pixel's channels): 3 % slower K1.
#ifndef TG_FG_MAX3
#define TG_FG_MAX3 1
#endif
template <bool kLow>
__device__ __forceinline__ uint32_t fg4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t b0,
                                        uint32_t b1, uint32_t b2, uint32_t t1) {
#if TG_FG_MAX3
  // |cur - prev| per byte, then each pixel's three channel differences into
  // the high bytes of 16-bit lanes (two pixels per word, one word per
  // channel; the low bytes only break ties) and one VIMNMX3.U16x2 per two
  // pixels: the 4 pixels' max difference, thresholded once.
  const uint32_t d0 = __vabsdiffu4(a0, b0), d1 = __vabsdiffu4(a1, b1), d2 = __vabsdiffu4(a2, b2);
  const uint32_t m01 = __vimax3_u16x2(__byte_perm(d0, d0, 0x3000), __byte_perm(d0, d1, 0x4010),
                                      __byte_perm(d0, d1, 0x5020));
  const uint32_t m23 = __vimax3_u16x2(__byte_perm(d1, d2, 0x5020), __byte_perm(d1, d2, 0x6030),
                                      __byte_perm(d1, d2, 0x7040));
  const uint32_t m = __byte_perm(m01, m23, 0x7531);
  return ((gt_bytes<kLow>(m, t1) & 0x80808080u) * 0x00204081u) >> 28;
#endif
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

// 32 pixels (96 bytes as 6 x 16) of cur/prev -> 32 raw foreground bits.
template <bool kLow>
__device__ __forceinline__ uint32_t fg_word(const uint4 (&c)[6], const uint4 (&p)[6], uint32_t t1) {
  uint32_t bits = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint4 c0 = c[3 * h], c1 = c[3 * h + 1], c2 = c[3 * h + 2];
    const uint4 p0 = p[3 * h], p1 = p[3 * h + 1], p2 = p[3 * h + 2];
    uint32_t v = fg4<kLow>(c0.x, c0.y, c0.z, p0.x, p0.y, p0.z, t1);
    v |= fg4<kLow>(c0.w, c1.x, c1.y, p0.w, p1.x, p1.y, t1) << 4;
    v |= fg4<kLow>(c1.z, c1.w, c2.x, p1.z, p1.w, p2.x, t1) << 8;
    v |= fg4<kLow>(c2.y, c2.z, c2.w, p2.y, p2.z, p2.w, t1) << 12;
    bits |= v << (16 * h);
  }
  return bits;
}

__device__ __forceinline__ void load96(uint4 (&v)[6], const uint8_t* p) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = lds128(p + 16 * k);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Walk of an item's frame chain: stages prev[f0], cur[f0], cur[f0+1], ...,
// with an extra prev[f] stage wherever prev[f] != cur[f-1].
struct Chain {
  int f, fend;
  bool need_prev;
  __device__ __forceinline__ bool done() const { return f >= fend && !need_prev; }
  // Source frame of the next stage; *out = frame index of the diff it
  // completes, or -1 for a chain start.
  __device__ __forceinline__ const uint8_t* next(const MaskArgs& a, int* out) {
    if (need_prev) {
      need_prev = false;
      *out = -1;
      return a.prev[f];
    }
    const uint8_t* p = a.cur[f];
    *out = f++;
    need_prev = f < fend && a.prev[f] != p;
    return p;
  }
};

struct ItemK1 {
  int f0, fend, y0;
};

__device__ __forceinline__ ItemK1 load_item(const MaskArgs& a, int item) {
  const int t = item % a.ntg, rb = item / a.ntg;
  ItemK1 it;
  it.f0 = t * a.kf;
  it.fend = min(a.n_frames, it.f0 + a.kf);
  it.y0 = rb * a.rows_per_item;
  return it;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused launch: K1b tasks (strip, frame, column group) in strip order, each
// after the K1 items that write its rows have published completion.
// Waits until the K1 items writing the rows of task t have published.
__device__ __forceinline__ void wait_dilate_task(const MaskArgs& a, int t, int lane) {
  const int sf = t / a.dgroups;
  const int f = sf % a.n_frames, sg = sf / a.n_frames;
  const int cy0 = sg * kK1bBands;
  const int y_lo = max(0, cy0 * kCell - a.radius);
  const int y_hi = min(a.H, (cy0 + kK1bBands) * kCell + a.radius) - 1;
  const int run = f / a.kf;
  for (int rb = y_lo / a.rows_per_item + lane; rb <= y_hi / a.rows_per_item; rb += 32) {
    const int rows = min(a.rows_per_item, a.H - rb * a.rows_per_item);
    const uint32_t want = static_cast<uint32_t>(kK1Group * a.nparts * rows);
    const uint32_t* flag = a.item_done + rb * a.ntg + run;
    while (ld_acquire(flag) < want) __nanosleep(256);
  }
}

// TG_K1_SPARSE_FUSED: the fused launch on the sparse bitmap too (K1 stores
// keep evict_last, K1b tasks read flags + flagged words through L2):
// config-2 step 1.959 -> 1.935 ms (same box), fused mask stage 1.250 ->
// 1.229 ms.
#ifndef TG_K1_SPARSE_FUSED
#define TG_K1_SPARSE_FUSED 1
#endif
constexpr bool kFusedSparse = TG_K1_SPARSE && TG_K1_SPARSE_FUSED;

__device__ __forceinline__ void run_dilate_task(const MaskArgs& a, int t, int lane) {
  __syncwarp();
  __threadfence();
  const int wi = t % a.dgroups, sf = t / a.dgroups;
  const int f = sf % a.n_frames, cy0 = sf / a.n_frames * kK1bBands;
  switch (a.radius) {
#define TG_DILATE_TASK(R) \
  case R:                 \
    if (a.d.mask_out)                                                          \
      dilate_strip<R, true, true, kFusedSparse>(a.d, f, cy0, wi, lane, nullptr); \
    else                                                                       \
      dilate_strip<R, true, false, kFusedSparse>(a.d, f, cy0, wi, lane, nullptr); \
    break;
    TG_DILATE_TASK(0) TG_DILATE_TASK(1) TG_DILATE_TASK(2) TG_DILATE_TASK(3) TG_DILATE_TASK(4)
    TG_DILATE_TASK(5) TG_DILATE_TASK(6) TG_DILATE_TASK(7) TG_DILATE_TASK(8)
#undef TG_DILATE_TASK
    default:
      break;
  }
}

// Drains the queue, waiting for each claimed task's items.
__device__ __forceinline__ void run_dilate_tasks(const MaskArgs& a, int lane) {
  for (;;) {
    int t = 0;
    if (lane == 0) t = static_cast<int>(atomicAdd(a.task_next, 1u));
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.n_tasks) return;
    wait_dilate_task(a, t, lane);
    run_dilate_task(a, t, lane);
  }
}

template <bool kLow>
__global__ void __launch_bounds__(kK1Threads, 1) mask_fg_kernel(const MaskArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int S = a.nslots;
  const int NS = kK1Groups * S;
  uint8_t* slots = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(NS) * a.slot_bytes);
  uint64_t* empty = full + NS;
  // frame whose diff a slot's row completes (-1: a chain start), written by
  // the producer before it arms the slot: consumers never read the pointer
  // tables
  int* slot_f = reinterpret_cast<int*>(empty + NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = a.rows_per_item * a.nparts;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kK1Group);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int part_bytes = a.part_words * 96;
  // K1 items go to the streaming CTAs; dedicated K1b CTAs (fused launch)
  // dilate the strips the stream has finished, on SMs of their own
  const int scta = static_cast<int>(blockIdx.x) - a.dctas, nscta = static_cast<int>(gridDim.x) - a.dctas;
  if (scta < 0) {
    run_dilate_tasks(a, lane);
    return;
  }
  const bool fused = a.item_done != nullptr;

  if (warp > kK1Groups * kK1Group) {  // K1b task warps (fused launch)
    if (fused) run_dilate_tasks(a, lane);
    return;
  }
  if (warp == kK1Groups * kK1Group) {
    // ===== producer: lane g streams group g's unit down the frame chain =====
    const int g = lane;
    const bool mine = g < units;
    uint32_t used = 0, fills = 0;  // per ring slot: filled before; fill-count parity
    int k = 0;                     // ring slot of the next stage
    for (int item = scta; item < a.total_items; item += nscta) {
      const ItemK1 it = load_item(a, item);
      const int row = it.y0 + g / a.nparts, part = g % a.nparts;
      const bool live = mine && row < a.H;
      const size_t off = static_cast<size_t>(row) * a.pitch + static_cast<size_t>(part) * part_bytes;
      const uint32_t bytes =
          static_cast<uint32_t>((min(part_bytes, a.rowbytes - part * part_bytes) + 15) & ~15);
      Chain ch{it.f0, it.fend, true};
      bool left = live;
      while (__any_sync(0xffffffffu, left)) {
        bool issued = false;
        if (left) {
          const int slot = g * S + k;
          const uint32_t bit = 1u << k;
          if (!(used & bit) || mbar_test_wait(&empty[slot], (fills & bit) ? 0u : 1u)) {
            int out;
            const uint8_t* src = ch.next(a, &out) + off;
            slot_f[slot] = out;
            mbar_arrive_expect_tx(&full[slot], bytes);
#if TG_K1_L2HINT & 1
            if (fused)
              bulk_g2s_hint(slots + static_cast<size_t>(slot) * a.slot_bytes, src, bytes,
                            &full[slot], l2_evict_first());
            else
#endif
              bulk_g2s(slots + static_cast<size_t>(slot) * a.slot_bytes, src, bytes, &full[slot]);
            used |= bit;
            fills ^= bit;
            if (++k == S) k = 0;
            issued = true;
            left = !ch.done();
          }
        }
        if (!__any_sync(0xffffffffu, issued)) __nanosleep(64);
      }
    }
    if (fused) run_dilate_tasks(a, lane);
    return;
  }

  // ===================== consumers ===========================================
  const uint32_t t1 =
      static_cast<uint32_t>(kLow ? a.threshold + 1 : a.threshold - 127) * 0x01010101u;
  const uint32_t lastmask = (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;
  const int g = warp / kK1Group;
  const int col = (warp - g * kK1Group) * 32 + lane;  // word within the part
  const bool in_slot = 96 * (col + 1) <= a.slot_bytes;  // lane's bytes inside a slot
  uint32_t fpar = 0;  // bit k: parity of the next full phase of ring slot k
  int k = 0;
  for (int item = scta; g < units && item < a.total_items; item += nscta) {
    const ItemK1 it = load_item(a, item);
    const int row = it.y0 + g / a.nparts, part = g % a.nparts;
    if (row >= a.H) continue;
    const int w = part * a.part_words + col;
    const bool valid = col < a.part_words && w < a.nwords;
    uint32_t* out = a.raw + static_cast<size_t>(row) * a.nwords + w;
    const size_t fstride = static_cast<size_t>(a.H) * a.nwords;
    const uint32_t keep = w == a.nwords - 1 ? lastmask : 0xffffffffu;
    // sparse: parts are 32-word aligned, so this warp's 32 words are one flag word
    const bool sparse = a.flags != nullptr;
    const int wbase = part * a.part_words + (warp - g * kK1Group) * 32;
    const bool fseg = (warp - g * kK1Group) * 32 < a.part_words && wbase < a.nwords;
    const int seg = wbase >> 5;
    // One stage: the next row of the chain into `cur`, diffed against `prv`
    // (the previous stage's row) unless it starts the chain.  The item ends
    // with frame fend-1 (a chain start never comes last); the two register
    // sets alternate, so rows never move between registers.
    auto stage = [&](uint4 (&cur)[6], const uint4 (&prv)[6]) -> int {
      const int slot = g * S + k;
      mbar_wait_sleep(&full[slot], (fpar >> k) & 1u);
      fpar ^= 1u << k;
      const int f = slot_f[slot];
      if (in_slot) load96(cur, slots + static_cast<size_t>(slot) * a.slot_bytes + 96 * col);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++k == S) k = 0;
      if (f >= 0) {
        const uint32_t fw = fg_word<kLow>(cur, prv, t1) & keep;
#if TG_K1_SPARSE
        if (sparse) {  // whole 8-word sectors holding a foreground bit + the row's flag word
          const uint32_t b = __ballot_sync(0xffffffffu, valid && fw != 0u);
          if (valid && ((b >> (lane & 24)) & 0xffu)) {
#if TG_K1_L2HINT & 2
            if (fused)
              st_hint(out + static_cast<size_t>(f) * fstride, fw, l2_evict_last());
            else
#endif
              out[static_cast<size_t>(f) * fstride] = fw;
          }
          if (lane == 0 && fseg) a.flags[(static_cast<size_t>(f) * a.H + row) * a.fwords + seg] = b;
          return f;
        }
#endif
#if TG_K1_L2HINT & 2
        if (valid) {
          if (fused)
            st_hint(out + static_cast<size_t>(f) * fstride, fw, l2_evict_last());
          else
            out[static_cast<size_t>(f) * fstride] = fw;
        }
#else
        if (valid) out[static_cast<size_t>(f) * fstride] = fw;
#endif
      }
      return f;
    };
    const int flast = it.fend - 1;
    uint4 A[6], B[6];
    for (;;) {
      if (stage(A, B) == flast) break;
      if (stage(B, A) == flast) break;
    }
    if (fused) {  // publish: this warp's raw words of the item are written
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(&a.item_done[item], 1u);
    }
  }
  if (fused) run_dilate_tasks(a, lane);
}

// ---- host launcher ---------------------------------------------------------
// Tuning overrides (probes only), read once per process.
static EnvInt g_env_slots{"TG_K1_SLOTS"}, g_env_runs{"TG_K1_RUNS"}, g_env_grid{"TG_K1_GRID"},
    g_env_dctas{"TG_K1_DCTAS"};
static SmemOptIn g_k1_smem[2];

static int env_or(EnvInt& e, int dflt) {
  const int v = e.get();
  return v >= 0 ? v : dflt;
}

static DilateArgs dilate_args(const uint32_t* d_raw, const uint32_t* d_zero, int W, int H,
                              uint32_t* d_cells,
                              uint32_t* d_active, uint32_t* d_mask) {
  DilateArgs d;
  d.raw = d_raw;
  d.zero = d_zero;
  d.flags = nullptr;
  d.fwords = 0;
  d.H = H;
  d.W = W;
  d.nwords = ceil_div(W, 32);
  d.cells_x = ceil_div(W, kCell);
  d.cells_y = ceil_div(H, kCell);
  d.act_words = ceil_div(d.cells_x, 32);
  d.cells = d_cells;
  d.active = d_active;
  d.mask_out = d_mask;
  return d;
}

// K1 work decomposition (items, ring slots) for one launch.
static cudaError_t plan_k1(MaskArgs& a, const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                           int n_frames, int W, int H, int pitch, int threshold, uint32_t* d_raw,
                           int sms, size_t* smem, uint32_t* d_flags = nullptr) {
  a = MaskArgs{};
  a.cur = d_cur;
  a.prev = d_prev;
  a.n_frames = n_frames;
  a.W = W;
  a.H = H;
  a.pitch = pitch;
  a.rowbytes = 3 * W;
  a.threshold = threshold;
  a.nwords = ceil_div(W, 32);
  a.nparts = ceil_div(a.nwords, kK1MaxPartWords);
  if (a.nparts > kK1Groups) return cudaErrorInvalidConfiguration;  // W > 16384
  a.part_words = ceil_div(a.nwords, a.nparts);
  if (d_flags) {  // sparse bitmap: 32-word aligned parts (one flag word per consumer warp)
    a.part_words = ceil_div(a.part_words, 32) * 32;
    a.nparts = ceil_div(a.nwords, a.part_words);
    a.flags = d_flags;
    a.fwords = ceil_div(a.nwords, 32);
  }
  a.rows_per_item = kK1Groups / a.nparts;
  a.nrb = ceil_div(H, a.rows_per_item);
  a.slot_bytes = (a.part_words * 96 + 127) & ~127;
  // per slot: the row, full + empty barriers, the stage's frame
  a.nslots = std::min(kK1MaxSlots, (kK1SmemBudget - 64) / (kK1Groups * (a.slot_bytes + 20)));
  a.nslots = std::max(2, std::min(a.nslots, env_or(g_env_slots, a.nslots)));
  // frame runs: enough items to balance the SMs
  int ntg = std::max(1, std::min(n_frames, ceil_div(8 * sms, a.nrb)));
  ntg = std::max(1, std::min(n_frames, env_or(g_env_runs, ntg)));
  a.kf = ceil_div(n_frames, ntg);
  a.ntg = ceil_div(n_frames, a.kf);
  a.total_items = a.ntg * a.nrb;
  a.raw = d_raw;
  *smem = static_cast<size_t>(kK1Groups) * a.nslots * (a.slot_bytes + 20);
  if (*smem > static_cast<size_t>(kK1SmemBudget)) return cudaErrorInvalidConfiguration;
  const bool low = threshold <= 127;
  return low ? g_k1_smem[1].ensure(mask_fg_kernel<true>, static_cast<int>(*smem))
             : g_k1_smem[0].ensure(mask_fg_kernel<false>, static_cast<int>(*smem));
}

cudaError_t launch_mask_fg(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                           int n_frames, int W, int H, int pitch, int threshold, uint32_t* d_raw,
                           uint32_t* d_flags, int sms, cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  MaskArgs a;
  size_t smem = 0;
  cudaError_t e =
      plan_k1(a, d_cur, d_prev, n_frames, W, H, pitch, threshold, d_raw, sms, &smem, d_flags);
  if (e != cudaSuccess) return e;
  int grid = std::min(a.total_items, sms);
  grid = std::max(1, std::min(a.total_items, env_or(g_env_grid, grid)));
  if (threshold <= 127)
    mask_fg_kernel<true><<<grid, kK1Threads, smem, stream>>>(a);
  else
    mask_fg_kernel<false><<<grid, kK1Threads, smem, stream>>>(a);
  return cudaGetLastError();
}

// The task queue head + item counters: total_items = runs x row blocks <=
// (8 sms / row blocks + 1) x row blocks <= 8 sms + H (plan_k1).
size_t mask_sync_words(int H, int sms) { return static_cast<size_t>(8) * sms + H + 2; }

cudaError_t launch_mask_fused(const uint8_t* const* d_cur, const uint8_t* const* d_prev,
                              int n_frames, int W, int H, int pitch, int threshold, int radius,
                              uint32_t* d_raw, const uint32_t* d_zero, uint32_t* d_flags,
                              uint32_t* d_cells, uint32_t* d_active, uint32_t* d_mask,
                              uint32_t* d_sync, int sms, cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  if (radius < 0 || radius > kMaxRadius) return cudaErrorInvalidValue;
  if (!kFusedSparse) d_flags = nullptr;
  MaskArgs a;
  size_t smem = 0;
  cudaError_t e =
      plan_k1(a, d_cur, d_prev, n_frames, W, H, pitch, threshold, d_raw, sms, &smem, d_flags);
  if (e != cudaSuccess) return e;
  a.d = dilate_args(d_raw, d_zero, W, H, d_cells, d_active, d_mask);
  a.d.flags = d_flags;
  a.d.fwords = a.fwords;
  if (a.d.act_words > kK1MaxActWords) return cudaErrorInvalidConfiguration;
  const size_t sync_words = mask_sync_words(H, sms);
  if (static_cast<size_t>(a.total_items) + 1 > sync_words) return cudaErrorInvalidConfiguration;
  a.radius = radius;
  a.dgroups = ceil_div(a.nwords, kK1GroupWords);
  a.strips = ceil_div(a.d.cells_y, kK1bBands);
  a.n_tasks = a.strips * n_frames * a.dgroups;
  a.task_next = d_sync;
  a.item_done = d_sync + 1;
  const size_t act_words = static_cast<size_t>(n_frames) * a.d.cells_y * a.d.act_words;
  if (d_active == d_sync + sync_words) {  // one allocation: one memset clears both
    e = cudaMemsetAsync(d_sync, 0, sizeof(uint32_t) * (sync_words + act_words), stream);
  } else {
    e = cudaMemsetAsync(d_sync, 0, sizeof(uint32_t) * (a.total_items + 1), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_active, 0, sizeof(uint32_t) * act_words, stream);
  }
  if (e != cudaSuccess) return e;
  // every CTA must be resident: task warps wait on items of other CTAs
  // Dedicated K1b CTAs: about 9 % of the SMs (the K1b share of the work),
  // rounded so every streaming CTA gets the same number of items -- the
  // stream then ends on all SMs at once (4K x 300: 1,620 items on 135 CTAs,
  // 13 K1b CTAs; mask stage 1.276 -> 1.255 ms, while 14 K1b CTAs leave some
  // streaming CTAs a 13th item: 1.306 ms).
  const int reserve = (sms * 9 + 50) / 100;
  const int per_cta = ceil_div(a.total_items, std::max(1, sms - reserve));
  const int streaming = ceil_div(a.total_items, per_cta);
  a.dctas = std::max(0, std::min(sms - 1, env_or(g_env_dctas, sms - streaming)));
  const int grid = std::min(a.total_items + a.dctas, sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kK1Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (threshold <= 127)
    e = cudaLaunchKernelEx(&cfg, mask_fg_kernel<true>, a);
  else
    e = cudaLaunchKernelEx(&cfg, mask_fg_kernel<false>, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_dilate_cells(const uint32_t* d_raw, const uint32_t* d_zero,
                                const uint32_t* d_flags, int n_frames,
                                int W, int H, int radius, uint32_t* d_cells, uint32_t* d_active,
                                uint32_t* d_mask, cudaStream_t stream) {
  if (n_frames <= 0) return cudaSuccess;
  DilateArgs d = dilate_args(d_raw, d_zero, W, H, d_cells, d_active, d_mask);
  d.flags = d_flags;
  d.fwords = ceil_div(d.nwords, 32);
  if (d.act_words > kK1MaxActWords) return cudaErrorInvalidConfiguration;
  const int dwarps = ceil_div(d.nwords, kK1GroupWords);
  const dim3 dg(n_frames * ceil_div(d.cells_y, kK1bBands)), db(dwarps * 32);
  switch (radius) {
#define TG_DILATE_CASE(R) \
  case R:                 \
    if (d_flags)          \
      dilate_cells_kernel<R, TG_K1_SPARSE != 0><<<dg, db, 0, stream>>>(d); \
    else                  \
      dilate_cells_kernel<R, false><<<dg, db, 0, stream>>>(d); \
    break;
    TG_DILATE_CASE(0) TG_DILATE_CASE(1) TG_DILATE_CASE(2) TG_DILATE_CASE(3) TG_DILATE_CASE(4)
    TG_DILATE_CASE(5) TG_DILATE_CASE(6) TG_DILATE_CASE(7) TG_DILATE_CASE(8)
#undef TG_DILATE_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tg
