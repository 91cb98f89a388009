// k_mask.cu -- K1: fused frame differencing + threshold + dilation +
// patch-grid occupancy (frozen spec DESIGN.md §3).
//
// The reference has no pixel stage (RoIs are inputs, trace.hpp:39-45); this
// kernel produces them.  Persistent, one CTA per SM, warp-specialized:
//
//  * 1 producer warp streams the rows of each work item -- (frame, segment of
//    up to 128 rows) plus r halo rows -- cur and prev side by side into a
//    ring of shared-memory slots with cp.async.bulk (the TMA bulk-copy
//    engine), full/empty mbarriers, no __syncthreads.  Items are walked in
//    frame-fastest order, so frame t's rows are read as `cur` by item (t, s)
//    and as `prev` by item (t+1, s) at about the same time and the second
//    read is an L2 hit.
//  * 8 consumer warps take stages round-robin; a lane turns 96 bytes (32 RGB
//    pixels) of cur/prev into one 32-bit raw-foreground word with packed
//    SIMD byte ops (VABSDIFF4 + SWAR compare + PRMT planar regroup) and
//    stores it in the item's bitmap in shared memory.
//  * When an item's bitmap is complete the consumers dilate it (vertical OR
//    over 2r+1 rows, horizontal funnel shifts with neighbour words taken from
//    adjacent lanes by shuffles) one 16-row cell band at a time and fold it
//    into per-cell popcounts and bbox bit-masks, written as packed u32 cell
//    summaries plus an activity bitmask.  Meanwhile the producer is already
//    prefetching the next item.
// HBM traffic is the frames themselves; the outputs are ~0.5% of it.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace tg {

// One consumer warp per smem slot (NS <= 8): a slot's consecutive phases are
// always waited on by the same warp, so mbarrier parity waits can never run
// two phases ahead.
constexpr int kK1MaxSlots = 8;
constexpr int kK1MaxThreads = 768;  // (NS*G + 1) warps; keeps <= 85 registers per thread
constexpr int kK1MaxSeg = 128;          // rows per work item (multiple of kCell)
constexpr int kK1SlotTarget = 24 * 1024;
constexpr int kK1SmemBudget = 227 * 1024;
constexpr int kK1GroupWords = 30;       // output words per warp task (lanes 1..30)
constexpr int kK1MaxBands = kK1MaxSeg / kCell;
constexpr int kK1MaxActWords = 16;      // act words per cell row held in smem (W <= 8192)

struct MaskArgs {
  const uint8_t* const* cur;
  const uint8_t* const* prev;
  int n_frames, W, H, pitch, rowbytes, threshold, radius;
  int nwords;          // ceil(W/32)
  int cells_x, cells_y, act_words;
  int rows_per_stage;  // RP
  int nstages;         // NS smem slots
  int group;           // G consumer warps per slot
  int seg_rows;        // SEG
  int nseg, total_items;
  uint32_t* cells;     // [F][cells_y][cells_x]
  uint32_t* active;    // [F][cells_y][act_words]
  uint32_t* mask_out;  // optional [F][H][nwords]
};

struct Item {
  int f, s0, s1, ya, yb, nst;
};

__device__ __forceinline__ Item load_item(const MaskArgs& a, int item) {
  Item it;
  it.f = item % a.n_frames;
  const int seg = item / a.n_frames;
  it.s0 = seg * a.seg_rows;
  it.s1 = min(a.H, it.s0 + a.seg_rows);
  it.ya = max(0, it.s0 - a.radius);
  it.yb = min(a.H, it.s1 + a.radius);
  it.nst = ceil_div(it.yb - it.ya, a.rows_per_stage);
  return it;
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
                                            uint32_t t1) {
  uint32_t bits = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && nbytes <= 48) break;
    const uint4 c0 = lds128(cs + 48 * h), c1 = lds128(cs + 48 * h + 16), c2 = lds128(cs + 48 * h + 32);
    const uint4 p0 = lds128(ps + 48 * h), p1 = lds128(ps + 48 * h + 16), p2 = lds128(ps + 48 * h + 32);
    uint32_t v = 0;
    v |= fg4<kLow>(c0.x, c0.y, c0.z, p0.x, p0.y, p0.z, t1);
    v |= fg4<kLow>(c0.w, c1.x, c1.y, p0.w, p1.x, p1.y, t1) << 4;
    v |= fg4<kLow>(c1.z, c1.w, c2.x, p1.z, p1.w, p2.x, t1) << 8;
    v |= fg4<kLow>(c2.y, c2.z, c2.w, p2.y, p2.z, p2.w, t1) << 12;
    bits |= v << (16 * h);
  }
  return bits;
}

__device__ __forceinline__ uint32_t pack_cell(int occ, uint32_t cols, uint32_t rows) {
  if (occ == 0) return 0u;
  const uint32_t x0 = __ffs(cols) - 1, x1 = 31 - __clz(cols);
  const uint32_t y0 = __ffs(rows) - 1, y1 = 31 - __clz(rows);
  return static_cast<uint32_t>(occ) | x0 << 9 | x1 << 13 | y0 << 17 | y1 << 21;
}

__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kK1MaxThreads, 1) mask_cells_kernel(const MaskArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int NS = a.nstages, RP = a.rows_per_stage;
  const int slot_bytes = 2 * RP * a.rowbytes;
  uint8_t* slots = smem;
  uint32_t* F = reinterpret_cast<uint32_t*>(smem + NS * slot_bytes);  // item bitmap
  const int f_rows = a.seg_rows + 2 * a.radius;
  uint32_t* act_s = F + f_rows * a.nwords;                          // [bands][act words]
  uint64_t* full = reinterpret_cast<uint64_t*>(act_s + kK1MaxBands * kK1MaxActWords);
  uint64_t* empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int G = a.group;       // consumer warps per slot
  const int ncw = NS * G;      // consumer warps; warp ncw is the producer
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kK1MaxBands * kK1MaxActWords; i += blockDim.x) act_s[i] = 0;
  __syncthreads();

  if (warp == ncw) {
    // ================= producer: one elected lane issues every copy =========
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 0;   // parity of the slot's current use
      bool wrapped = false; // every slot used once already
      for (int item = blockIdx.x; item < a.total_items; item += gridDim.x) {
        const Item it = load_item(a, item);
        const uint8_t* cur = a.cur[it.f];
        const uint8_t* prev = a.prev[it.f];
        for (int st = 0; st < it.nst; ++st) {
          if (wrapped) mbar_wait(&empty[slot], phase ^ 1u);  // previous use released
          const int y0 = it.ya + st * RP;
          const int nr = min(RP, it.yb - y0);
          const uint32_t bytes = static_cast<uint32_t>(nr * a.rowbytes);
          uint8_t* dc = slots + slot * slot_bytes;
          uint8_t* dp = dc + RP * a.rowbytes;
          const uint8_t* sc = cur + static_cast<size_t>(y0) * a.pitch;
          const uint8_t* sp = prev + static_cast<size_t>(y0) * a.pitch;
          mbar_arrive_expect_tx(&full[slot], 2 * bytes);
          if (a.pitch == a.rowbytes) {
            bulk_g2s(dc, sc, bytes, &full[slot]);
            bulk_g2s(dp, sp, bytes, &full[slot]);
          } else {
            for (int k = 0; k < nr; ++k) {
              bulk_g2s(dc + k * a.rowbytes, sc + static_cast<size_t>(k) * a.pitch, a.rowbytes,
                       &full[slot]);
              bulk_g2s(dp + k * a.rowbytes, sp + static_cast<size_t>(k) * a.pitch, a.rowbytes,
                       &full[slot]);
            }
          }
          if (++slot == NS) {
            slot = 0;
            phase ^= 1u;
            wrapped = true;
          }
        }
      }
    }
    return;
  }

  // ===================== consumers ===========================================
  const bool t_low = a.threshold <= 127;
  const uint32_t t1 =
      static_cast<uint32_t>(t_low ? a.threshold + 1 : a.threshold - 127) * 0x01010101u;
  const uint32_t lastmask = (a.W & 31) ? ((1u << (a.W & 31)) - 1u) : 0xffffffffu;
  const int ngroups = ceil_div(a.nwords, kK1GroupWords);
  const int my_slot = warp / G, sub = warp - my_slot * G;
  // Stages are dealt to slots round-robin; this warp group owns every NS-th
  // stage.  first_st: this group's first stage within the current item;
  // phase: parity of its slot's next use.
  int first_st = my_slot;
  uint32_t phase = 0;
  for (int item = blockIdx.x; item < a.total_items; item += gridDim.x) {
    const Item it = load_item(a, item);
    // ---- raw foreground words: this group's stages of the item ----
    int st = first_st;
    for (; st < it.nst; st += NS) {
      const int slot = my_slot;
      mbar_wait(&full[slot], phase);
      phase ^= 1u;
      const int y0 = it.ya + st * RP;
      const int nr = min(RP, it.yb - y0);
      const uint8_t* sc = slots + slot * slot_bytes;
      const uint8_t* sp = sc + RP * a.rowbytes;
      for (int k = 0; k < nr; ++k) {
        uint32_t* frow = F + (y0 + k - it.ya) * a.nwords;
        for (int w = sub * 32 + lane; w < a.nwords; w += 32 * G) {
          const int off = 96 * w;
          const int nbytes = min(96, a.rowbytes - off);
          const uint8_t* cw = sc + k * a.rowbytes + off;
          const uint8_t* pw = sp + k * a.rowbytes + off;
          uint32_t fw = t_low ? fg_word<true>(cw, pw, nbytes, t1) : fg_word<false>(cw, pw, nbytes, t1);
          if (w == a.nwords - 1) fw &= lastmask;
          frow[w] = fw;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // slot may be refilled
    }
    first_st = st - it.nst;  // stages continue into the next item
    consumer_bar(ncw * 32);  // bitmap of the item complete

    // ---- dilation + cell summaries, one (16-row band, 30-word group) task
    //      per warp at a time ----
    const int nbands = ceil_div(it.s1 - it.s0, kCell);
    for (int task = warp; task < nbands * ngroups; task += ncw) {
      const int band = task / ngroups, grp = task - band * ngroups;
      const int w = grp * kK1GroupWords + lane - 1;
      const bool col_ok = w >= 0 && w < a.nwords;
      const bool owns = lane >= 1 && lane <= kK1GroupWords && col_ok;
      const int yb0 = it.s0 + band * kCell;
      const int yb1 = min(yb0 + kCell, it.s1);
      int occ_lo = 0, occ_hi = 0;
      uint32_t col_lo = 0, col_hi = 0, row_lo = 0, row_hi = 0;
      for (int y = yb0; y < yb1; ++y) {
        uint32_t v = 0;
        if (col_ok) {
          const int lo = max(y - a.radius, it.ya), hi = min(y + a.radius, it.yb - 1);
          for (int yy = lo; yy <= hi; ++yy) v |= F[(yy - it.ya) * a.nwords + w];
        }
        const uint32_t vm = __shfl_up_sync(0xffffffffu, v, 1);
        const uint32_t vp = __shfl_down_sync(0xffffffffu, v, 1);
        uint32_t d = v;
        for (int k = 1; k <= a.radius; ++k)
          d |= __funnelshift_r(v, vp, k) | __funnelshift_l(vm, v, k);
        if (w == a.nwords - 1) d &= lastmask;
        if (!owns) d = 0;
        if (a.mask_out && owns) a.mask_out[(static_cast<size_t>(it.f) * a.H + y) * a.nwords + w] = d;
        const uint32_t dl = d & 0xffffu, dh = d >> 16;
        const int ly = y - yb0;
        occ_lo += __popc(dl);
        occ_hi += __popc(dh);
        col_lo |= dl;
        col_hi |= dh;
        row_lo |= (dl ? 1u : 0u) << ly;
        row_hi |= (dh ? 1u : 0u) << ly;
      }
      if (owns) {
        const int cy = yb0 / kCell, cx = 2 * w;
        const size_t cbase = (static_cast<size_t>(it.f) * a.cells_y + cy) * a.cells_x;
        a.cells[cbase + cx] = pack_cell(occ_lo, col_lo, row_lo);
        if (cx + 1 < a.cells_x) a.cells[cbase + cx + 1] = pack_cell(occ_hi, col_hi, row_hi);
        const uint32_t bits = (occ_lo > 0 ? 1u : 0u) | (occ_hi > 0 ? 2u : 0u);
        if (bits) atomicOr(&act_s[band * kK1MaxActWords + (cx >> 5)], bits << (cx & 31));
      }
    }
    consumer_bar(ncw * 32);  // act_s complete, bitmap free for the next item
    for (int i = threadIdx.x; i < nbands * a.act_words; i += ncw * 32) {
      const int band = i / a.act_words, aw = i - band * a.act_words;
      const int cy = (it.s0 / kCell) + band;
      a.active[(static_cast<size_t>(it.f) * a.cells_y + cy) * a.act_words + aw] =
          act_s[band * kK1MaxActWords + aw];
      act_s[band * kK1MaxActWords + aw] = 0;
    }
    // act_s is next touched after the next item's first consumer_bar().
  }
}

// ---- host launcher ---------------------------------------------------------
struct MaskPlan {
  int rows_per_stage, nstages, seg_rows;
  size_t smem;
};

static MaskPlan plan_mask(int W, int radius) {
  const int rowbytes = 3 * W, nwords = ceil_div(W, 32);
  MaskPlan p;
  p.rows_per_stage = std::max(1, std::min(8, kK1SlotTarget / (2 * rowbytes)));
  const size_t slot = static_cast<size_t>(2) * p.rows_per_stage * rowbytes;
  const size_t fixed = static_cast<size_t>(kK1MaxBands) * kK1MaxActWords * 4 + 2 * 8 * 8 + 128;
  p.nstages = kK1MaxSlots;
  if (const char* e = std::getenv("TG_K1_SLOTS")) p.nstages = std::max(2, std::min(kK1MaxSlots, std::atoi(e)));
  p.seg_rows = kK1MaxSeg;
  auto total = [&](int ns, int seg) {
    return fixed + ns * slot + static_cast<size_t>(seg + 2 * radius) * nwords * 4;
  };
  const size_t budget = static_cast<size_t>(kK1SmemBudget);
  while (total(p.nstages, p.seg_rows) > budget && p.nstages > 4) --p.nstages;
  while (total(p.nstages, p.seg_rows) > budget && p.seg_rows > 64) p.seg_rows -= kCell;
  while (total(p.nstages, p.seg_rows) > budget && p.nstages > 2) --p.nstages;
  while (total(p.nstages, p.seg_rows) > budget && p.seg_rows > kCell) p.seg_rows -= kCell;
  p.smem = total(p.nstages, p.seg_rows);
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
  const MaskPlan mp = plan_mask(W, radius);
  if (mp.smem > static_cast<size_t>(kK1SmemBudget) || a.act_words > kK1MaxActWords)
    return cudaErrorInvalidConfiguration;
  a.rows_per_stage = mp.rows_per_stage;
  a.nstages = mp.nstages;
  // consumer warps per slot: enough lanes for a stage's words, within the
  // thread budget
  int G = std::min(4, std::max(1, ceil_div(a.nwords, 32)));
  if (const char* gs = std::getenv("TG_K1_GROUP")) G = std::max(1, std::atoi(gs));
  while (G > 1 && (mp.nstages * G + 1) * 32 > kK1MaxThreads) --G;
  a.group = G;
  a.seg_rows = mp.seg_rows;
  a.nseg = ceil_div(H, a.seg_rows);
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
  mask_cells_kernel<<<grid, (mp.nstages * a.group + 1) * 32, mp.smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace tg
