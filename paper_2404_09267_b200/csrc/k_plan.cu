// k_plan.cu -- per-frame planner (K2 RoI boxes + K3 partition + K4 stitch
// plan), the frame-order scan, and the drop-in rect-level kernels.
//
// K2 (absent from the reference): 8-connected components over
// the active patch-grid cells by union-find on 16-bit labels in shared
// memory (atomic-CAS min linking, so every root is its component's first
// cell in raster order), then one pixel-tight box per component from the
// per-cell bboxes K1 wrote.  Boxes are ranked by their root cell, i.e. in
// the oracle's raster order.
// K3 = partition() (partition.hpp:119-143) and K4 = stitch_all()
// (stitch.hpp:108-146) on that frame's admitted patches (sim.hpp:262,
// 302-332), both from rect_core.cuh.  The planner finally emits the gather
// jobs: every placement plus every final free rect, which tile each canvas
// exactly, grouped by canvas.
#include <algorithm>

#include "kernels.cuh"
#include "rect_core.cuh"

namespace tg {

constexpr int kPlanThreads = 512;

__device__ __forceinline__ int uf_find(volatile uint16_t* L, int x) {
  int p = L[x];
  while (p != x) {
    x = p;
    p = L[x];
  }
  return x;
}

__device__ __forceinline__ void uf_merge(uint16_t* L, int a, int b) {
  volatile uint16_t* VL = L;
  while (true) {
    a = uf_find(VL, a);
    b = uf_find(VL, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    // Link root a (larger) under b: 16-bit atomic min via CAS.
    unsigned short old = VL[a];
    while (old > b) {
      const unsigned short prev =
          atomicCAS(reinterpret_cast<unsigned short*>(&L[a]), old, static_cast<unsigned short>(b));
      if (prev == old) break;
      old = prev;
    }
    if (old == a) return;  // a was still a root and now points at b
    a = old;               // someone re-linked a meanwhile: retry from there
  }
}

__device__ __forceinline__ bool act_bit(const uint32_t* act, int aw, int cy, int cx) {
  return (act[cy * aw + (cx >> 5)] >> (cx & 31)) & 1u;
}

// Block-wide exclusive scan of n ints in place (n <= any), returns total.
__device__ int block_exclusive_scan(int* v, int n, int* warp_tmp) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  int carry = 0;
  for (int base = 0; base < n; base += nt) {
    const int i = base + tid;
    const int x = i < n ? v[i] : 0;
    int s = x;
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
      warp_tmp[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const int before = (wid ? warp_tmp[wid - 1] : 0) + s - x;
    const int total = warp_tmp[nt / 32 - 1];
    __syncthreads();
    if (i < n) v[i] = carry + before;
    carry += total;
  }
  __syncthreads();
  return carry;
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ ZoneAcc zacc;
  __shared__ tg_patch_meta spatch[kMaxZones];
  __shared__ int adm_w[kMaxZones], adm_h[kMaxZones], adm_idx[kMaxZones];
  __shared__ FreeRect freel[2 * kMaxZones + 2];
  __shared__ StitchOut souts[kMaxZones];
  __shared__ int warp_tmp[32];
  __shared__ int s_nrois;

  const int f = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int aw = a.act_words, ncw = a.cells_y * aw, cx_n = a.cells_x;
  uint32_t* act = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* rootm = act + ncw;
  int* wpre = reinterpret_cast<int*>(rootm + ncw);
  int* bx0 = wpre + ncw + 1;
  int* by0 = bx0 + a.max_rois;
  int* bx1 = by0 + a.max_rois;
  int* by1 = bx1 + a.max_rois;
  uint16_t* L = reinterpret_cast<uint16_t*>(by1 + a.max_rois);

  const uint32_t* gact = a.active + static_cast<size_t>(f) * ncw;
  const uint32_t* gcells = a.cells + static_cast<size_t>(f) * a.cells_y * cx_n;

  // ---- K2: labels on active cells --------------------------------------
  for (int i = tid; i < ncw; i += nt) {
    const uint32_t bits = gact[i];
    act[i] = bits;
    uint32_t m = bits;
    const int cy = i / aw, cxb = (i - cy * aw) * 32;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int idx = cy * cx_n + cxb + b;
      L[idx] = static_cast<uint16_t>(idx);
    }
  }
  __syncthreads();
  for (int i = tid; i < ncw; i += nt) {
    uint32_t m = act[i];
    const int cy = i / aw, cxb = (i - cy * aw) * 32;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int cx = cxb + b, idx = cy * cx_n + cx;
      if (cx > 0 && act_bit(act, aw, cy, cx - 1)) uf_merge(L, idx, idx - 1);
      if (cy > 0) {
        if (cx > 0 && act_bit(act, aw, cy - 1, cx - 1)) uf_merge(L, idx, idx - cx_n - 1);
        if (act_bit(act, aw, cy - 1, cx)) uf_merge(L, idx, idx - cx_n);
        if (cx + 1 < cx_n && act_bit(act, aw, cy - 1, cx + 1)) uf_merge(L, idx, idx - cx_n + 1);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < ncw; i += nt) {
    uint32_t m = act[i], roots = 0;
    const int cy = i / aw, cxb = (i - cy * aw) * 32;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int idx = cy * cx_n + cxb + b;
      const int r = uf_find(L, idx);
      if (r == idx) roots |= 1u << b;
    }
    rootm[i] = roots;
    wpre[i] = __popc(roots);
  }
  __syncthreads();
  // Full path compression (separate pass: finds above must see stable roots).
  for (int i = tid; i < ncw; i += nt) {
    uint32_t m = act[i];
    const int cy = i / aw, cxb = (i - cy * aw) * 32;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int idx = cy * cx_n + cxb + b;
      L[idx] = static_cast<uint16_t>(uf_find(L, idx));
    }
  }
  const int ncomp = block_exclusive_scan(wpre, ncw, warp_tmp);
  if (tid == 0) {
    wpre[ncw] = ncomp;
    int n = ncomp;
    if (n > a.max_rois) {
      raise_error(a.err, TG_ERR_CAPACITY, kErrRoiCapacity, f, ncomp, a.max_rois);
      n = a.max_rois;
    }
    s_nrois = n;
  }
  __syncthreads();
  const int nr = s_nrois;
  for (int r = tid; r < nr; r += nt) {
    bx0[r] = INT_MAX;
    by0[r] = INT_MAX;
    bx1[r] = INT_MIN;
    by1[r] = INT_MIN;
  }
  __syncthreads();
  for (int i = tid; i < ncw; i += nt) {
    uint32_t m = act[i];
    const int cy = i / aw, cxb = (i - cy * aw) * 32;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int cx = cxb + b, idx = cy * cx_n + cx;
      const int root = L[idx];
      const int rcy = root / cx_n, rcx = root - rcy * cx_n;
      const int rw = rcy * aw + (rcx >> 5);
      const int rank = wpre[rw] + __popc(rootm[rw] & ((1u << (rcx & 31)) - 1u));
      if (rank >= nr) continue;
      const uint32_t v = gcells[idx];
      atomicMin(&bx0[rank], cx * kCell + static_cast<int>(v >> 9 & 15u));
      atomicMax(&bx1[rank], cx * kCell + static_cast<int>(v >> 13 & 15u));
      atomicMin(&by0[rank], cy * kCell + static_cast<int>(v >> 17 & 15u));
      atomicMax(&by1[rank], cy * kCell + static_cast<int>(v >> 21 & 15u));
    }
  }
  __syncthreads();
  tg_rect* frois = a.rois + static_cast<size_t>(f) * a.max_rois;
  for (int r = tid; r < nr; r += nt)
    frois[r] = tg_rect{bx0[r], by0[r], bx1[r] - bx0[r] + 1, by1[r] - by0[r] + 1};
  const int nz = a.X * a.Y;
  zone_acc_init(zacc, nz, tid, nt);
  if (tid == 0) a.n_rois[f] = nr;
  __syncthreads();

  // ---- K3: partition (Alg. 1) ------------------------------------------
  partition_accumulate(frois, nr, a.W, a.H, a.X, a.Y, zacc, a.err, f, nullptr, tid, nt);
  __syncthreads();
  if (tid >= 32) return;
  const int lane = tid;
  const int np = partition_emit(zacc, nz, a.frame_ids[f], a.gen_us[f], a.slo_us, a.bpp, 0, spatch,
                                lane);
  __syncwarp();
  // Admission (sim.hpp:262): w <= M && h <= N; rejected patches keep their
  // ids but are never stitched.
  int na = 0;
  for (int jb = 0; jb < np; jb += 32) {
    const int j = jb + lane;
    const bool ok = j < np && spatch[j].rect.w <= a.M && spatch[j].rect.h <= a.N;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (j < np) {
      a.patches[static_cast<size_t>(f) * nz + j] = spatch[j];
      a.admitted[static_cast<size_t>(f) * nz + j] = ok ? 1 : 0;
    }
    if (ok) {
      const int k = na + __popc(m & ((1u << lane) - 1u));
      adm_w[k] = spatch[j].rect.w;
      adm_h[k] = spatch[j].rect.h;
      adm_idx[k] = j;
    }
    na += __popc(m);
  }
  for (int j = np + lane; j < nz; j += 32) a.admitted[static_cast<size_t>(f) * nz + j] = 0;
  __syncwarp();

  // ---- K4: stitch plan (Alg. 2 solver) ---------------------------------
  int nfree = 0;
  const int nc = na ? bssf_stitch(adm_w, adm_h, nullptr, na, a.M, a.N, freel, 2 * kMaxZones + 2,
                                  souts, &nfree, a.err, f, lane)
                    : 0;
  __syncwarp();
  if (lane == 0) {
    a.n_patches[f] = np;
    a.n_placements[f] = na;
    a.n_canvases[f] = nc < 0 ? 0 : nc;
  }
  if (nc <= 0) return;
  tg_placement* fpl = a.placements + static_cast<size_t>(f) * nz;
  for (int k = lane; k < na; k += 32) {
    tg_placement p;
    p.patch_id = static_cast<uint64_t>(adm_idx[k]);  // frame-local; the scan makes it global
    p.canvas_index = souts[k].canvas;
    p.position = tg_rect{souts[k].x, souts[k].y, adm_w[k], adm_h[k]};
    p.reserved = 0;
    fpl[k] = p;
  }
  // Gather jobs grouped by canvas: placements (queue order) then free rects.
  Job* fj = a.jobs + static_cast<size_t>(f) * a.job_cap;
  uint32_t* fcj = a.canvas_jobs + static_cast<size_t>(f) * nz;
  const int nitems = na + nfree;
  int pos = 0;
  for (int c = 0; c < nc; ++c) {
    const int start = pos;
    for (int ib = 0; ib < nitems; ib += 32) {
      const int it = ib + lane;
      bool mine = false;
      Job jb{};
      if (it < na) {
        mine = souts[it].canvas == c;
        const tg_rect src = spatch[adm_idx[it]].rect;
        jb = Job{static_cast<uint16_t>(souts[it].x), static_cast<uint16_t>(souts[it].y),
                 static_cast<uint16_t>(src.w), static_cast<uint16_t>(src.h), f,
                 static_cast<uint16_t>(src.x), static_cast<uint16_t>(src.y)};
      } else if (it < nitems) {
        const FreeRect fr = freel[it - na];
        mine = fr.canvas == c;
        jb = Job{static_cast<uint16_t>(fr.x), static_cast<uint16_t>(fr.y),
                 static_cast<uint16_t>(fr.w), static_cast<uint16_t>(fr.h), -1,
                 static_cast<uint16_t>(fr.seq & 0xffff), static_cast<uint16_t>(fr.seq >> 16)};
      }
      const unsigned m = __ballot_sync(0xffffffffu, mine);
      if (mine) fj[pos + __popc(m & ((1u << lane) - 1u))] = jb;
      pos += __popc(m);
    }
    if (lane == 0) fcj[c] = static_cast<uint32_t>(start) | static_cast<uint32_t>(pos - start) << 16;
  }
}

// ---- frame-order scan: global patch ids and canvas numbering -------------
__global__ void __launch_bounds__(1024) scan_kernel(const ScanArgs a) {
  __shared__ long long wtmp_p[32], wtmp_c[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
  // ~0 = continue numbering where the previous run on this pipeline ended
  // (streaming chunks without a host round trip).
  const uint64_t first_id = a.first_id == ~0ull ? *a.id_state : a.first_id;
  __syncthreads();
  long long run_p = 0, run_c = 0;
  for (int base = 0; base < a.n_frames; base += nt) {
    const int f = base + tid;
    const long long vp = f < a.n_frames ? a.n_patches[f] : 0;
    const long long vc = f < a.n_frames ? a.n_canvases[f] : 0;
    long long sp = vp, sc = vc;
    for (int o = 1; o < 32; o <<= 1) {
      const long long yp = __shfl_up_sync(0xffffffffu, sp, o);
      const long long yc = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) {
        sp += yp;
        sc += yc;
      }
    }
    if (lane == 31) {
      wtmp_p[wid] = sp;
      wtmp_c[wid] = sc;
    }
    __syncthreads();
    if (wid == 0) {
      long long tp = lane < nt / 32 ? wtmp_p[lane] : 0, tc = lane < nt / 32 ? wtmp_c[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long yp = __shfl_up_sync(0xffffffffu, tp, o);
        const long long yc = __shfl_up_sync(0xffffffffu, tc, o);
        if (lane >= o) {
          tp += yp;
          tc += yc;
        }
      }
      wtmp_p[lane] = tp;
      wtmp_c[lane] = tc;
    }
    __syncthreads();
    const long long pb = run_p + (wid ? wtmp_p[wid - 1] : 0) + sp - vp;
    const long long cb = run_c + (wid ? wtmp_c[wid - 1] : 0) + sc - vc;
    if (f < a.n_frames) {
      const uint64_t id0 = first_id + static_cast<uint64_t>(pb);
      tg_patch_meta* fp = a.patches + static_cast<size_t>(f) * a.zones;
      for (int j = 0; j < vp; ++j) fp[j].patch_id = id0 + static_cast<uint64_t>(j);
      tg_placement* fl = a.placements + static_cast<size_t>(f) * a.zones;
      for (int k = 0; k < a.n_placements[f]; ++k) fl[k].patch_id = id0 + fl[k].patch_id;
      a.canvas_base[f] = cb;
      for (int c = 0; c < vc; ++c)
        if (cb + c < a.max_canvases)
          a.canvas_map[cb + c] = static_cast<uint32_t>(f) << 6 | static_cast<uint32_t>(c);
    }
    run_p += wtmp_p[nt / 32 - 1];
    run_c += wtmp_c[nt / 32 - 1];
    __syncthreads();
  }
  if (tid == 0) {
    *a.id_state = first_id + static_cast<uint64_t>(run_p);
    a.canvas_base[a.n_frames] = run_c;
    long long total = run_c;
    if (total > a.max_canvases) {
      raise_error(a.err, TG_ERR_CAPACITY, kErrCanvasCapacity, total, a.max_canvases);
      total = a.max_canvases;
    }
    *a.gather_units = static_cast<int32_t>(total * a.nbands);
  }
}

// ---- drop-in / batched rect-level kernels ---------------------------------
// One block per frame: partition() of host-supplied RoIs.
__global__ void __launch_bounds__(256) partition_batch_kernel(const PartitionBatchArgs a) {
  __shared__ ZoneAcc zacc;
  __shared__ tg_patch_meta sp[kMaxZones];
  const int f = blockIdx.x, tid = threadIdx.x, nz = a.X * a.Y;
  const tg_frame_spec fs = a.frames[f];
  const int r0 = a.roi_offsets[f], r1 = a.roi_offsets[f + 1];
  zone_acc_init(zacc, nz, tid, blockDim.x);
  __syncthreads();
  partition_accumulate(a.rois + r0, r1 - r0, fs.width, fs.height, a.X, a.Y, zacc, a.err, f,
                       a.zone_of ? a.zone_of + r0 : nullptr, tid, blockDim.x);
  __syncthreads();
  if (tid >= 32) return;
  const int np = partition_emit(zacc, nz, fs.frame_id, fs.generation_time_us, fs.slo_us, a.bpp,
                                a.first_ids[f], sp, tid);
  __syncwarp();
  for (int j = tid; j < np; j += 32) a.patches[static_cast<size_t>(f) * nz + j] = sp[j];
  if (tid == 0) a.n_patches[f] = np;
}

// One warp per queue; the free set lives in global workspace.
__global__ void __launch_bounds__(128) stitch_batch_kernel(const StitchBatchArgs a) {
  const int q = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (q >= a.n_queues) return;
  const int o0 = a.offsets[q], n = a.offsets[q + 1] - o0;
  int* pw = a.dims_ws + 5 * o0;
  int* ph = pw + n;
  StitchOut* so = reinterpret_cast<StitchOut*>(ph + n);
  uint64_t* ids = a.ids_ws + o0;
  for (int i = lane; i < n; i += 32) {
    pw[i] = a.queue[o0 + i].rect.w;
    ph[i] = a.queue[o0 + i].rect.h;
    ids[i] = a.queue[o0 + i].patch_id;
  }
  __syncwarp();
  FreeRect* fl = a.free_ws + 2 * o0 + q;
  int nfree = 0;
  const int nc = bssf_stitch(pw, ph, ids, n, a.M, a.N, fl, 2 * n + 1, so, &nfree, a.err, q, lane);
  __syncwarp();
  if (nc >= 0) {
    for (int i = lane; i < n; i += 32) {
      tg_placement p;
      p.patch_id = ids[i];
      p.canvas_index = so[i].canvas;
      p.position = tg_rect{so[i].x, so[i].y, pw[i], ph[i]};
      p.reserved = 0;
      a.placements[o0 + i] = p;
    }
  }
  if (lane == 0) {
    a.n_canvases[q] = nc;
    if (a.n_free) a.n_free[q] = nfree;
  }
}

// ---- launchers --------------------------------------------------------------
size_t plan_smem_bytes(int cells_x, int cells_y, int max_rois) {
  const int aw = ceil_div(cells_x, 32);
  const size_t ncw = static_cast<size_t>(cells_y) * aw;
  return ncw * 4 * 2 + (ncw + 1) * 4 + static_cast<size_t>(max_rois) * 16 +
         static_cast<size_t>(cells_x) * cells_y * 2 + 16;
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream) {
  if (a.n_frames <= 0) return cudaSuccess;
  const size_t smem = plan_smem_bytes(a.cells_x, a.cells_y, a.max_rois);
  cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  plan_kernel<<<a.n_frames, kPlanThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream) {
  scan_kernel<<<1, 1024, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_partition_batch(const PartitionBatchArgs& a, cudaStream_t stream) {
  if (a.n_frames <= 0) return cudaSuccess;
  partition_batch_kernel<<<a.n_frames, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stitch_batch(const StitchBatchArgs& a, cudaStream_t stream) {
  if (a.n_queues <= 0) return cudaSuccess;
  const int per_block = 4;
  stitch_batch_kernel<<<ceil_div(a.n_queues, per_block), 32 * per_block, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace tg
