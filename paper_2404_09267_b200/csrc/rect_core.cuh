// rect_core.cuh -- device restatement of the reference's rect-level core:
// Alg. 1 partition (partition.hpp:69-143) and Alg. 2's patch-stitching
// solver (stitch.hpp:66-146), shared by the fused per-frame planner and the
// drop-in / batched entry points.
#pragma once

#include <climits>

#include "common.cuh"

namespace tg {

// make_zones (partition.hpp:69-88): row-major from the bottom-left, the last
// column/row absorbs the remainder.
__device__ __forceinline__ tg_rect zone_rect(int z, int W, int H, int X, int Y) {
  const int zw = W / X, zh = H / Y;
  const int row = z / X, col = z - row * X;
  tg_rect r;
  r.x = col * zw;
  r.y = row * zh;
  r.w = (col == X - 1) ? W - r.x : zw;
  r.h = (row == Y - 1) ? H - r.y : zh;
  return r;
}

// overlap_area (geometry.hpp:44-49), int64.
__device__ __forceinline__ long long overlap_area(const tg_rect& a, const tg_rect& b) {
  const int ow = min(a.x + a.w, b.x + b.w) - max(a.x, b.x);
  const int oh = min(a.y + a.h, b.y + b.h) - max(a.y, b.y);
  if (ow <= 0 || oh <= 0) return 0;
  return static_cast<long long>(ow) * static_cast<long long>(oh);
}

// assign_rois (partition.hpp:93-112): zone of maximum overlap, strict '>'
// so ties keep the lowest zone index; -1 if the RoI misses the frame.
// Only the zones in the RoI's column and row span can overlap it (zone c
// covers [c*zw, (c+1)*zw), the last one up to W), and visiting them in
// row-major order keeps the reference's tie rule.
__device__ __forceinline__ int best_zone(const tg_rect& r, int W, int H, int X, int Y) {
  const int zw = W / X, zh = H / Y;  // >= 1: finer grids are rejected up front
  const int xe = r.x + r.w - 1, ye = r.y + r.h - 1;
  const int c0 = r.x <= 0 ? 0 : min(r.x / zw, X - 1), c1 = xe <= 0 ? 0 : min(xe / zw, X - 1);
  const int r0 = r.y <= 0 ? 0 : min(r.y / zh, Y - 1), r1 = ye <= 0 ? 0 : min(ye / zh, Y - 1);
  long long best = 0;
  int bz = -1;
  for (int row = r0; row <= r1; ++row) {
    for (int col = c0; col <= c1; ++col) {
      const int z = row * X + col;
      const long long s = overlap_area(r, zone_rect(z, W, H, X, Y));
      if (s > best) {
        best = s;
        bz = z;
      }
    }
  }
  return bz;
}

// Per-zone enclosing-rect accumulators in shared memory (Z zones at most).
template <int Z>
struct ZoneAccT {
  int x0[Z], y0[Z], x1[Z], y1[Z], cnt[Z];
};
using ZoneAcc = ZoneAccT<kMaxZones>;

template <class ZA>
__device__ __forceinline__ void zone_acc_init(ZA& z, int nz, int tid, int nthreads) {
  for (int i = tid; i < nz; i += nthreads) {
    z.x0[i] = INT_MAX;
    z.y0[i] = INT_MAX;
    z.x1[i] = INT_MIN;
    z.y1[i] = INT_MIN;
    z.cnt[i] = 0;
  }
}

// Block-cooperative assignment of n RoIs into the zone accumulators.
// Returns nothing; an RoI outside the frame latches kErrRoiOutside.
template <class RectAt, class ZA>
__device__ __forceinline__ void partition_accumulate_at(RectAt rect_at, int n, int W, int H,
                                                        int X, int Y, ZA& z, DevError* err,
                                                        int frame, int* zone_of, int tid,
                                                        int nthreads) {
  for (int i = tid; i < n; i += nthreads) {
    const tg_rect r = rect_at(i);
    const int bz = best_zone(r, W, H, X, Y);
    if (zone_of) zone_of[i] = bz;
    if (bz < 0) {
      // With zone_of the caller reports the FIRST bad index itself (the
      // reference throws at the lowest one, partition.hpp:106-108).
      if (!zone_of) raise_error(err, TG_ERR_INVALID_ARGUMENT, kErrRoiOutside, i, frame);
      continue;
    }
    atomicMin(&z.x0[bz], r.x);
    atomicMin(&z.y0[bz], r.y);
    atomicMax(&z.x1[bz], r.x + r.w);
    atomicMax(&z.y1[bz], r.y + r.h);
    atomicAdd(&z.cnt[bz], 1);
  }
}

__device__ __forceinline__ void partition_accumulate(const tg_rect* rois, int n, int W, int H,
                                                     int X, int Y, ZoneAcc& z, DevError* err,
                                                     int frame, int* zone_of, int tid,
                                                     int nthreads) {
  partition_accumulate_at([rois](int i) { return rois[i]; }, n, W, H, X, Y, z, err, frame, zone_of,
                          tid, nthreads);
}

// One warp: one patch per non-empty zone in zone order (partition.hpp:
// 125-141).  patch_id = first_id + rank; returns the patch count.
template <class ZA>
__device__ __forceinline__ int partition_emit(const ZA& z, int nz, uint64_t frame_id,
                                              int64_t gen_us, int64_t slo_us, double bpp,
                                              uint64_t first_id, tg_patch_meta* out, int lane) {
  int base = 0;
  for (int zb = 0; zb < nz; zb += 32) {
    const int zi = zb + lane;
    const bool ne = zi < nz && z.cnt[zi] > 0;
    const unsigned m = __ballot_sync(0xffffffffu, ne);
    if (ne) {
      const int rank = base + __popc(m & ((1u << lane) - 1u));
      tg_patch_meta p;
      p.patch_id = first_id + static_cast<uint64_t>(rank);
      p.source_frame_id = frame_id;
      p.rect.x = z.x0[zi];
      p.rect.y = z.y0[zi];
      p.rect.w = z.x1[zi] - z.x0[zi];
      p.rect.h = z.y1[zi] - z.y0[zi];
      p.generation_time_us = gen_us;
      p.slo_us = slo_us;
      p.deadline_us = gen_us + slo_us;
      p.size_bytes = static_cast<int64_t>(
          ceil(static_cast<double>(static_cast<long long>(p.rect.w) * p.rect.h) * bpp));
      out[rank] = p;
    }
    base += __popc(m);
  }
  return base;
}

// ---- Alg. 2 patch-stitching solver, one warp ------------------------------
// Best-short-side fit over every live free rect of every open canvas;
// ties by lower canvas, then lower y, then lower x (candidate_better,
// stitch.hpp:72-81) -- a total order because a canvas's free rects are
// disjoint, so a lexicographic min over two 64-bit keys, (score, canvas) then
// (y, x), finds the reference's choice for any canvas count (scores,
// coordinates < 2^16: canvas sides are bounded by 65535 at the ABI).  The
// free set is kept unordered (swap-remove); each rect carries its insertion
// seq so the reference's list order can be rebuilt.  Guillotine split per
// stitch.hpp:86-99.  dims(i) -> int2 (w, h) and id(i) read the queue;
// emit(i, canvas, x, y) receives each placement (lane 0).  Returns the canvas
// count, or -1 after latching an error (oversize patch / free capacity).
struct StitchOut {
  int canvas;
  int x, y;
};

template <class Dims, class Id, class Emit>
__device__ __forceinline__ int bssf_stitch_q(Dims dims, Id id, Emit emit, int n, int M, int N,
                                             FreeRect* fl, int cap, int* n_free_out, DevError* err,
                                             int queue, int lane) {
  int nfree = 0, nc = 0, seq = 0;
  for (int i = 0; i < n; ++i) {
    const int2 d = dims(i);
    const int w = d.x, h = d.y;
    if (w > M || h > N) {
      if (lane == 0)
        raise_error(err, TG_ERR_INVALID_ARGUMENT, kErrPatchOversize,
                    static_cast<long long>(id(i)), w, h, queue);
      return -1;
    }
    unsigned long long b1 = ~0ull, b2 = ~0ull;
    int bi = -1;
    for (int k = lane; k < nfree; k += 32) {
      const FreeRect c = fl[k];
      if (c.w < w || c.h < h) continue;
      const unsigned s = static_cast<unsigned>(min(c.w - w, c.h - h));
      const unsigned long long k1 = (static_cast<unsigned long long>(s) << 32) |
                                    static_cast<unsigned long long>(static_cast<unsigned>(c.canvas));
      const unsigned long long k2 = (static_cast<unsigned long long>(c.y) << 32) |
                                    static_cast<unsigned long long>(static_cast<unsigned>(c.x));
      if (k1 < b1 || (k1 == b1 && k2 < b2)) {
        b1 = k1;
        b2 = k2;
        bi = k;
      }
    }
    const unsigned long long g1 = warp_min_u64(b1);
    const unsigned long long g2 = warp_min_u64(b1 == g1 ? b2 : ~0ull);
    FreeRect chosen;
    const bool fits = g1 != ~0ull;
    if (!fits) {  // nothing fits: open a blank canvas (stitch.hpp:129-135)
      chosen = FreeRect{0, 0, M, N, nc, -1};
      ++nc;
    } else {
      const unsigned owner = __ballot_sync(0xffffffffu, b1 == g1 && b2 == g2 && bi >= 0);
      const int src = __ffs(owner) - 1;
      bi = __shfl_sync(0xffffffffu, bi, src);
      chosen = fl[bi];
    }
    __syncwarp();
    const int lw = chosen.w - w, lh = chosen.h - h;
    FreeRect a, b;
    if (lw <= lh) {
      a = FreeRect{chosen.x + w, chosen.y, lw, chosen.h, chosen.canvas, 0};
      b = FreeRect{chosen.x, chosen.y + h, w, lh, chosen.canvas, 0};
    } else {
      a = FreeRect{chosen.x + w, chosen.y, lw, h, chosen.canvas, 0};
      b = FreeRect{chosen.x, chosen.y + h, chosen.w, lh, chosen.canvas, 0};
    }
    const bool keep_a = a.w > 0 && a.h > 0, keep_b = b.w > 0 && b.h > 0;
    int nf = nfree;
    if (fits) --nf;  // swap-remove the chosen rect
    const int need = nf + (keep_a ? 1 : 0) + (keep_b ? 1 : 0);
    if (need > cap) {
      if (lane == 0) raise_error(err, TG_ERR_CAPACITY, kErrFreeCapacity, queue, cap);
      return -1;
    }
    if (lane == 0) {
      if (fits) fl[bi] = fl[nfree - 1];
      if (keep_a) {
        a.seq = seq++;
        fl[nf++] = a;
      }
      if (keep_b) {
        b.seq = seq++;
        fl[nf++] = b;
      }
      emit(i, chosen.canvas, chosen.x, chosen.y);
    } else {
      seq += (keep_a ? 1 : 0) + (keep_b ? 1 : 0);
      nf += (keep_a ? 1 : 0) + (keep_b ? 1 : 0);
    }
    nfree = nf;
    __syncwarp();
  }
  if (n_free_out) *n_free_out = nfree;
  return nc;
}

// Queue in shared arrays (the per-frame planner).
__device__ __forceinline__ int bssf_stitch(const int* pw, const int* ph, const uint64_t* pid,
                                           int n, int M, int N, FreeRect* fl, int cap,
                                           StitchOut* out, int* n_free_out, DevError* err,
                                           int queue, int lane) {
  return bssf_stitch_q([pw, ph](int i) { return make_int2(pw[i], ph[i]); },
                       [pid](int i) { return pid ? pid[i] : static_cast<uint64_t>(i); },
                       [out](int i, int c, int x, int y) { out[i] = StitchOut{c, x, y}; }, n, M, N,
                       fl, cap, n_free_out, err, queue, lane);
}

}  // namespace tg
