// ccl.cuh -- K2: 8-connected components over the active patch-grid cells
// of one frame, one CTA, everything in shared memory.
//
// Run-based union-find: a horizontal run of active cells is labelled by its
// head (bit tricks on the activity bitmask, no atomics), so unions are only
// needed between runs of adjacent rows that touch diagonally or vertically.
// A run's label slot is (its activity word) * 16 + (its ordinal among the
// word's run heads): a word holds at most 16 heads, slots are in raster
// order, and the label array is 16 u16 per 32 cells instead of one per cell
// (small enough for three planner CTAs per SM).  Links always point from the
// larger to the smaller slot (16-bit atomic-CAS min), so every root is its
// component's first run in raster order -- the oracle's component order
// (orc_extract_rois).  Finds use path halving.  Each run then folds its
// pixel-tight extent (from the cell summaries K1b wrote) into its
// component's box.
#pragma once

#include <climits>

#include "common.cuh"

namespace tg {

// First cell of the run containing set bit x of a cell row.
__device__ __forceinline__ int run_start(const uint32_t* row, int x) {
  int wi = x >> 5;
  const uint32_t zeros = ~row[wi] & ((1u << (x & 31)) - 1u);
  if (zeros) return (wi << 5) + (32 - __clz(zeros));
  for (--wi; wi >= 0; --wi) {
    const uint32_t nz = ~row[wi];
    if (nz) return (wi << 5) + (32 - __clz(nz));
  }
  return 0;
}

// Last cell of the run containing set bit x.
__device__ __forceinline__ int run_end(const uint32_t* row, int x, int aw) {
  int wi = x >> 5;
  const uint32_t zeros = ~row[wi] & ~((2u << (x & 31)) - 1u);
  if (zeros) return (wi << 5) + __ffs(zeros) - 2;
  for (++wi; wi < aw; ++wi) {
    const uint32_t z = ~row[wi];
    if (z) return (wi << 5) + __ffs(z) - 2;
  }
  return aw * 32 - 1;
}

__device__ __forceinline__ int uf_find(uint16_t* L, int x) {
  volatile uint16_t* V = L;
  int p = V[x];
  while (p != x) {
    const int gp = V[p];
    if (gp != p) V[x] = static_cast<uint16_t>(gp);  // path halving (ancestor store)
    x = p;
    p = gp;
  }
  return x;
}

// Read-only find, for the passes after the unions: a halving store there
// could overwrite another thread's freshly compressed root pointer with a
// non-root ancestor.
__device__ __forceinline__ int uf_find_ro(const uint16_t* L, int x) {
  const volatile uint16_t* V = L;
  int p = V[x];
  while (p != x) {
    x = p;
    p = V[x];
  }
  return x;
}

__device__ __forceinline__ void uf_merge(uint16_t* L, int a, int b) {
  volatile uint16_t* V = L;
  while (true) {
    a = uf_find(L, a);
    b = uf_find(L, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    unsigned short old = V[a];  // atomic min(L[a], b) via 16-bit CAS
    while (old > b) {
      const unsigned short prev =
          atomicCAS(reinterpret_cast<unsigned short*>(&L[a]), old, static_cast<unsigned short>(b));
      if (prev == old) break;
      old = prev;
    }
    if (old == a) return;  // a was a root and now hangs under b
    a = old;               // a was re-linked concurrently: continue from its new parent
  }
}

// Head bits of a word: set bits whose left neighbour (bit-1, or bit 31 of the
// previous word of the same row) is clear.
__device__ __forceinline__ uint32_t run_heads(const uint32_t* row, int wi) {
  const uint32_t w = row[wi];
  const uint32_t carry = wi > 0 ? row[wi - 1] >> 31 : 0u;
  return w & ~((w << 1) | carry);
}

// Block-wide exclusive scan of n ints in place; returns the total.  One
// pass: thread t owns the contiguous chunk [t*k, t*k + k), k = ceil(n / nt),
// so the block needs two barriers however large n is (ncw = 1,080 words at
// 4K: 3 per thread).
__device__ int block_exclusive_scan(int* v, int n, int* warp_tmp) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int k = (n + nt - 1) / nt;
  const int i0 = min(n, tid * k), i1 = min(n, i0 + k);
  int own = 0;
  for (int i = i0; i < i1; ++i) own += v[i];
  int s = own;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += y;
  }
  if (lane == 31) warp_tmp[wid] = s;
  __syncthreads();
  if (wid == 0) {
    int t = lane < nt / 32 ? warp_tmp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tmp[lane] = t;
  }
  __syncthreads();
  int run = (wid ? warp_tmp[wid - 1] : 0) + s - own;
  const int total = warp_tmp[nt / 32 - 1];
  for (int i = i0; i < i1; ++i) {
    const int x = v[i];
    v[i] = run;
    run += x;
  }
  __syncthreads();
  return total;
}

#ifdef TG_PLAN_PHASES  // diagnostics build: per-phase clock64 marks of thread 0
#define TG_PH(i) do { if (threadIdx.x == 0) tg_ph_mark[i] = clock64(); } while (0)
#else
#define TG_PH(i) do { } while (0)
#endif

constexpr int kHeadsPerWord = 16;  // run heads in a 32-cell activity word

struct CclSmem {
  uint32_t* act;    // [ncw] activity bits (copied from K1b's bitmask)
  uint32_t* rootm;  // [ncw] root runs, by head ordinal within the word
  int* wpre;        // [ncw + 1] exclusive prefix of popc(rootm)
  int *bx0, *by0, *bx1, *by1;  // [max_rois]
  uint16_t* L;      // [ncw * 16] run labels by slot
};

// Slot of the run whose head is bit b of activity word `word` (index wi of
// its row `row`).
__device__ __forceinline__ int head_slot(const uint32_t* row, int wi, int word, int b) {
  return word * kHeadsPerWord + __popc(run_heads(row, wi) & ((1u << b) - 1u));
}

// Returns the number of RoIs (components), boxes in bx0..by1 (inclusive
// pixel bounds), ranked by root cell.  Latches kErrRoiCapacity and clamps.
__device__ int ccl_frame(const uint32_t* gact, const uint32_t* gcells, int cx_n, int cy_n,
                         int max_rois, const CclSmem& s, int* warp_tmp, int* s_n, DevError* err,
                         int frame
#ifdef TG_PLAN_PHASES
                         , long long* tg_ph_mark
#endif
                         ) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int aw = ceil_div(cx_n, 32), ncw = cy_n * aw;
  for (int i = tid; i < ncw; i += nt) s.act[i] = gact[i];
  __syncthreads();
  TG_PH(1);
  // labels of run heads
  for (int i = tid; i < ncw; i += nt) {
    const int cy = i / aw, wi = i - cy * aw;
    const int nh = __popc(run_heads(s.act + cy * aw, wi));
    for (int k = 0; k < nh; ++k) s.L[i * kHeadsPerWord + k] = static_cast<uint16_t>(i * kHeadsPerWord + k);
  }
  __syncthreads();
  TG_PH(2);
  // unions between each run and the runs it touches in the row above
  for (int i = tid; i < ncw; i += nt) {
    const int cy = i / aw, wi = i - cy * aw;
    if (cy == 0) continue;
    const uint32_t* row = s.act + cy * aw;
    const uint32_t* up = row - aw;
    uint32_t h = run_heads(row, wi);
    for (int k = 0; h; ++k) {
      const int b = __ffs(h) - 1;
      h &= h - 1;
      const int a0 = (wi << 5) + b;
      const int e = run_end(row, a0, aw);
      const int head = i * kHeadsPerWord + k;
      int x = max(a0 - 1, 0);
      const int xe = min(e + 1, cx_n - 1);
      while (x <= xe) {
        int uw = x >> 5;
        uint32_t m = up[uw] & (~0u << (x & 31));
        while (!m && ++uw <= (xe >> 5)) m = up[uw];
        if (!m) break;
        x = (uw << 5) + __ffs(m) - 1;
        if (x > xe) break;
        const int us = run_start(up, x);
        uf_merge(s.L, head, head_slot(up, us >> 5, i - aw - wi + (us >> 5), us & 31));
        x = run_end(up, x, aw) + 2;
      }
    }
  }
  __syncthreads();
  TG_PH(3);
  // roots, and every head's label compressed to its root in the same pass:
  // the unions are over, so a stored root is final and concurrent finds
  // through this slot just arrive sooner
  for (int i = tid; i < ncw; i += nt) {
    const int cy = i / aw, wi = i - cy * aw;
    const int nh = __popc(run_heads(s.act + cy * aw, wi));
    uint32_t roots = 0;
    for (int k = 0; k < nh; ++k) {
      const int sl = i * kHeadsPerWord + k;
      const int r = uf_find_ro(s.L, sl);
      if (r == sl) roots |= 1u << k;
      else s.L[sl] = static_cast<uint16_t>(r);
    }
    s.rootm[i] = roots;
    s.wpre[i] = __popc(roots);
  }
  __syncthreads();
  TG_PH(4);
  const int ncomp = block_exclusive_scan(s.wpre, ncw, warp_tmp);
  if (tid == 0) {
    s.wpre[ncw] = ncomp;
    int n = ncomp;
    if (n > max_rois) {
      raise_error(err, TG_ERR_CAPACITY, kErrRoiCapacity, frame, ncomp, max_rois);
      n = max_rois;
    }
    *s_n = n;
  }
  __syncthreads();
  const int nr = *s_n;
  for (int r = tid; r < nr; r += nt) {
    s.bx0[r] = INT_MAX;
    s.by0[r] = INT_MAX;
    s.bx1[r] = INT_MIN;
    s.by1[r] = INT_MIN;
  }
  __syncthreads();
  TG_PH(5);
  // Boxes.  x: every run's end cells.  y: only the component's top cell row
  // (its root's row) can hold the box's top pixel and only its bottom row the
  // bottom one, so just those runs scan their cells' y extents.  Pass 1 also
  // raises by1 to 16 * (bottom cell row); pass 2 keeps it in [16 * row,
  // 16 * row + 15], so by1 >> 4 names the bottom row throughout.
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = tid; i < ncw; i += nt) {
      const int cy = i / aw, wi = i - cy * aw;
      const uint32_t* row = s.act + cy * aw;
      uint32_t h = run_heads(row, wi);
      for (int k = 0; h; ++k) {
        const int b = __ffs(h) - 1;
        h &= h - 1;
        const int a0 = (wi << 5) + b;
        const int e = run_end(row, a0, aw);
        const int root = s.L[i * kHeadsPerWord + k];
        const int rw = root / kHeadsPerWord, ro = root - rw * kHeadsPerWord;
        const int rank = s.wpre[rw] + __popc(s.rootm[rw] & ((1u << ro) - 1u));
        if (rank >= nr) continue;
        const uint32_t* crow = gcells + static_cast<size_t>(cy) * cx_n;
        if (pass == 0) {
          const uint32_t va = __ldg(crow + a0), ve = __ldg(crow + e);
          atomicMin(&s.bx0[rank], a0 * kCell + static_cast<int>(va >> 9 & 15u));
          atomicMax(&s.bx1[rank], e * kCell + static_cast<int>(ve >> 13 & 15u));
          atomicMax(&s.by1[rank], cy * kCell);
          continue;
        }
        const bool top = rw / aw == cy, bottom = (s.by1[rank] >> 4) == cy;
        if (!top && !bottom) continue;
        // y extent over the run's cell summaries: eight loads in flight per step
        int y0 = INT_MAX, y1 = INT_MIN;
        int cx = a0;
        for (; cx + 8 <= e + 1; cx += 8) {
          uint32_t v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = __ldg(crow + cx + t);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            y0 = min(y0, static_cast<int>(v[t] >> 17 & 15u));
            y1 = max(y1, static_cast<int>(v[t] >> 21 & 15u));
          }
        }
        for (; cx <= e; ++cx) {
          const uint32_t v = __ldg(crow + cx);
          y0 = min(y0, static_cast<int>(v >> 17 & 15u));
          y1 = max(y1, static_cast<int>(v >> 21 & 15u));
        }
        if (top) atomicMin(&s.by0[rank], cy * kCell + y0);
        if (bottom) atomicMax(&s.by1[rank], cy * kCell + y1);
      }
    }
    __syncthreads();
    TG_PH(6 + pass);
  }
  __syncthreads();
  return nr;
}

}  // namespace tg
