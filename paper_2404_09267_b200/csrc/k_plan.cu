// k_plan.cu -- per-frame planner (K2 RoI boxes + K3 partition + K4 stitch
// plan), the frame-order scan, and the drop-in rect-level kernels.
//
// One CTA per frame:
//   K2 (absent from the reference): ccl.cuh -- 8-connected
//      components over the active cells, one pixel-tight box per component
//      in the oracle's raster order;
//   K3 partition() (partition.hpp:119-143) and admission (sim.hpp:262);
//   K4 stitch_all() (stitch.hpp:108-146) on the frame's admitted patches
//      (sim.hpp:302-332), one warp;
// then the gather jobs: every placement plus every final free rect, which
// tile each canvas exactly, grouped by canvas and sorted
// by x so the gather can walk canvas rows left to right.
#include <algorithm>

#include "ccl.cuh"
#include "kernels.cuh"
#include "rect_core.cuh"

namespace tg {

constexpr int kPlanThreads = 256;

// Rank sort of one canvas's jobs by (dx, dy) -- unique, since a canvas's
// placements and free rects are disjoint -- from tmp into out.  One warp.
__device__ __forceinline__ void sort_jobs_by_x(const Job* tmp, int n, Job* out, int lane) {
  for (int i = lane; i < n; i += 32) {
    const Job a = tmp[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const Job b = tmp[j];
      rank += (b.dx < a.dx) || (b.dx == a.dx && (b.dy < a.dy || (b.dy == a.dy && j < i)));
    }
    out[rank] = a;
  }
}

// K3/K4 working set; aliases the K2 (CCL) region of dynamic smem once the
// RoI boxes are out, so three planner CTAs fit on an SM.
struct PlanTail {
  tg_patch_meta spatch[kMaxZones];
  FreeRect freel[2 * kMaxZones + 2];
  StitchOut souts[kMaxZones];
  Job sjobs[3 * kMaxZones];
};

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ ZoneAcc zacc;
  __shared__ int adm_w[kMaxZones], adm_h[kMaxZones], adm_idx[kMaxZones];
  __shared__ int warp_tmp[32];
  __shared__ int s_nrois;
  PlanTail& T = *reinterpret_cast<PlanTail*>(dsm);
  tg_patch_meta* spatch = T.spatch;
  FreeRect* freel = T.freel;
  StitchOut* souts = T.souts;
  Job* sjobs = T.sjobs;

  const int f = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int cx_n = a.cells_x, cy_n = a.cells_y, aw = a.act_words, ncw = cy_n * aw;
  CclSmem cs;
  cs.act = reinterpret_cast<uint32_t*>(dsm);
  cs.rootm = cs.act + ncw;
  cs.wpre = reinterpret_cast<int*>(cs.rootm + ncw);
  cs.bx0 = cs.wpre + ncw + 1;
  cs.by0 = cs.bx0 + a.max_rois;
  cs.bx1 = cs.by0 + a.max_rois;
  cs.by1 = cs.bx1 + a.max_rois;
  cs.L = reinterpret_cast<uint16_t*>(cs.by1 + a.max_rois);

  // ---- K2: RoI boxes ---------------------------------------------------------
  const int nr = ccl_frame(a.active + static_cast<size_t>(f) * ncw,
                           a.cells + static_cast<size_t>(f) * cy_n * cx_n, cx_n, cy_n, a.max_rois,
                           cs, warp_tmp, &s_nrois, a.err, f);
  tg_rect* frois = a.rois + static_cast<size_t>(f) * a.max_rois;
  for (int r = tid; r < nr; r += nt)
    frois[r] = tg_rect{cs.bx0[r], cs.by0[r], cs.bx1[r] - cs.bx0[r] + 1, cs.by1[r] - cs.by0[r] + 1};
  const int nz = a.X * a.Y;
  zone_acc_init(zacc, nz, tid, nt);
  if (tid == 0) a.n_rois[f] = nr;
  __syncthreads();

  // ---- K3: partition (Alg. 1) --------------------------------------------
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

  // ---- K4: stitch plan (Alg. 2 solver) -------------------------------------
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
  // Gather jobs: placements and free rects grouped by canvas, sorted by x.
  Job* fj = a.jobs + static_cast<size_t>(f) * a.job_cap;
  uint32_t* fcj = a.canvas_jobs + static_cast<size_t>(f) * nz;
  const int nitems = na + nfree;
  int pos = 0;
  for (int c = 0; c < nc; ++c) {
    int cnt = 0;
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
      if (mine) sjobs[cnt + __popc(m & ((1u << lane) - 1u))] = jb;
      cnt += __popc(m);
    }
    __syncwarp();
    sort_jobs_by_x(sjobs, cnt, fj + pos, lane);
    __syncwarp();
    if (lane == 0) fcj[c] = static_cast<uint32_t>(pos) | static_cast<uint32_t>(cnt) << 16;
    pos += cnt;
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
      const uint32_t* fcj = a.canvas_jobs + static_cast<size_t>(f) * a.zones;
      for (int c = 0; c < vc; ++c)
        if (cb + c < a.max_canvases)
          a.ranges[cb + c] = make_uint2(static_cast<uint32_t>(f) * a.job_cap + (fcj[c] & 0xffffu),
                                        fcj[c] >> 16);
    }
    run_p += wtmp_p[nt / 32 - 1];
    run_c += wtmp_c[nt / 32 - 1];
    __syncthreads();
  }
  if (tid == 0) {
    *a.id_state = first_id + static_cast<uint64_t>(run_p);
    a.canvas_base[a.n_frames] = run_c;
    long long total = run_c;
    if (a.max_canvases == 0) {
      total = 0;  // planning only: per-frame canvases are not materialized
    } else if (total > a.max_canvases) {
      raise_error(a.err, TG_ERR_CAPACITY, kErrCanvasCapacity, total, a.max_canvases);
      total = a.max_canvases;
    }
    a.gather_units[0] = static_cast<int32_t>(total * a.nbands);
    a.gather_units[1] = 0;  // K5's claim counters
    a.gather_units[2] = 0;
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
  const size_t ccl = ncw * 4 * 2 + (ncw + 1) * 4 + static_cast<size_t>(max_rois) * 16 +
                     ncw * kHeadsPerWord * 2 + 16;
  return ccl > sizeof(PlanTail) ? ccl : sizeof(PlanTail);
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
