// k_plan.cu -- per-frame planner (K2 RoI boxes + K3 partition + K4 stitch
// plan) with the frame-order prefix, and the drop-in rect-level kernels.
//
// One CTA per frame:
//   K2 (absent from the reference): ccl.cuh -- 8-connected
//      components over the active cells, one pixel-tight box per component
//      in the oracle's raster order;
//   K3 partition() (partition.hpp:119-143) and admission (sim.hpp:262);
//   K4 stitch_all() (stitch.hpp:108-146) on the frame's admitted patches
//      (sim.hpp:302-332), one warp;
// then the frame-order prefix of patch and canvas counts (global patch ids,
// sim.hpp:249-251, and canvas numbering) by decoupled look-back between the
// frames' CTAs -- frames are taken from a ticket counter, so every
// predecessor of a frame is already running -- and the gather jobs: every
// placement plus every final free rect, which tile each canvas exactly
// (SURVEY Appendix P5), grouped by canvas and sorted by x so the gather can
// walk canvas rows left to right.  The CTA of the last frame leaves the
// totals (canvas count, K5 units, next patch id) in device memory.
#include <algorithm>

#include "ccl.cuh"
#include "kernels.cuh"
#include "rect_core.cuh"

namespace tg {

#ifndef TG_PLAN_THREADS
#define TG_PLAN_THREADS 512  // 3 CTAs per SM still fit (300 4K frames: one wave); 256: 0.066 ms, 512: 0.052
#endif
constexpr int kPlanThreads = TG_PLAN_THREADS;

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


// ---- look-back words: epoch(16) | flag(2) | patches(23) | canvases(23) -----
// flag 1: this frame's own counts, 2: inclusive prefix through this frame.
// A word from an earlier launch carries another epoch and reads as absent.
constexpr uint32_t kLookAgg = 1, kLookIncl = 2;
constexpr uint64_t kLookMask = (1ull << 23) - 1;

__device__ __forceinline__ uint64_t look_pack(uint32_t epoch, uint32_t flag, uint64_t p, uint64_t c) {
  return static_cast<uint64_t>(epoch & 0xffffu) << 48 | static_cast<uint64_t>(flag) << 46 |
         (p & kLookMask) << 23 | (c & kLookMask);
}

__device__ __forceinline__ void st_release64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_volatile32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Warp 0 of frame f's CTA publishes (np, nc) as soon as K4 has them
// (look_publish), builds its gather jobs, then resolves the exclusive prefix
// over frames 0..f-1 (look_back) -- the wait for slower predecessors hides
// behind the job sort.
__device__ __forceinline__ void look_publish(const PlanArgs& a, int f, uint32_t epoch, uint64_t np,
                                             uint64_t nc, int lane) {
  if (lane == 0) st_release64(&a.look[f], look_pack(epoch, f == 0 ? kLookIncl : kLookAgg, np, nc));
}

// after look_publish: sums the predecessors back to the nearest inclusive
// prefix and publishes this frame's
__device__ void look_back(const PlanArgs& a, int f, uint32_t epoch, uint64_t np, uint64_t nc,
                          uint64_t* ex_p, uint64_t* ex_c, int lane) {
  uint64_t sp = 0, sc = 0;
  for (int j = f - 1; j >= 0; j -= 32) {
    const int idx = j - lane;
    uint64_t v = 0;
    uint32_t flag = 0;
    if (idx >= 0) {
      for (;;) {
        v = ld_acquire64(&a.look[idx]);
        flag = static_cast<uint32_t>(v >> 46) & 3u;
        if ((v >> 48) == (epoch & 0xffffu) && flag != 0) break;
        __nanosleep(64);
      }
    }
    const unsigned incl = __ballot_sync(0xffffffffu, flag == kLookIncl);
    const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest predecessor with a prefix
    uint64_t vp = (idx >= 0 && lane <= stop) ? (v >> 23) & kLookMask : 0;
    uint64_t vc = (idx >= 0 && lane <= stop) ? v & kLookMask : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vp += __shfl_xor_sync(0xffffffffu, vp, o);
      vc += __shfl_xor_sync(0xffffffffu, vc, o);
    }
    sp += vp;
    sc += vc;
    if (incl) break;
  }
  if (lane == 0 && f > 0) st_release64(&a.look[f], look_pack(epoch, kLookIncl, sp + np, sc + nc));
  *ex_p = sp;
  *ex_c = sc;
}

// Totals of the run, by the CTA that saw the inclusive prefix of the last frame.
__device__ void plan_totals(const PlanArgs& a, uint64_t first_id, uint64_t total_p,
                            long long total_c) {
  *a.id_state = first_id + total_p;
  a.canvas_base[a.n_frames] = total_c;
  long long total = total_c;
  if (a.max_canvases == 0) {
    total = 0;  // planning only: per-frame canvases are not materialized
  } else if (total > a.max_canvases) {
    raise_error(a.err, TG_ERR_CAPACITY, kErrCanvasCapacity, total, a.max_canvases);
    total = a.max_canvases;
  }
  a.gather_units[0] = static_cast<int32_t>(total * a.nbands);
  a.gather_units[1] = 0;  // K5's claim counters
  a.gather_units[2] = 0;
  if (a.desc_head) {
    const long long np = static_cast<long long>(total_p);
    if (np > a.desc_cap) raise_error(a.err, TG_ERR_CAPACITY, kErrDescCapacity, np, a.desc_cap);
    a.desc_head->count = np < a.desc_cap ? np : a.desc_cap;
    a.desc_head->cap = a.desc_cap;
  }
}

// K3/K4 working set; aliases the K2 (CCL) region of dynamic smem once the
// RoI boxes are out, so three planner CTAs fit on an SM.
template <int Z>
struct PlanTail {
  tg_patch_meta spatch[Z];
  FreeRect freel[2 * Z + 2];
  StitchOut souts[Z];
  Job sjobs[3 * Z];
};

#ifdef TG_PLAN_PHASES
__device__ unsigned long long g_plan_phase[16];
#endif

// Z: zones per frame at most (kMaxZones, or kMaxPlanZones for finer grids)
template <int Z>
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ ZoneAccT<Z> zacc;
  __shared__ int adm_w[Z], adm_h[Z], adm_idx[Z];
  __shared__ int warp_tmp[32];
  __shared__ int s_nrois;
  PlanTail<Z>& T = *reinterpret_cast<PlanTail<Z>*>(dsm);
  tg_patch_meta* spatch = T.spatch;
  FreeRect* freel = T.freel;
  StitchOut* souts = T.souts;
  Job* sjobs = T.sjobs;

  __shared__ int s_f;
  __shared__ uint32_t s_epoch;
  __shared__ unsigned long long s_first;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) {
    s_epoch = ld_volatile32(&a.psync[2]);
    s_first = a.first_id == ~0ull ? *reinterpret_cast<const volatile uint64_t*>(a.id_state)
                                   : a.first_id;
    // frames in ticket order: a frame's predecessors are all running or done,
    // so its look-back cannot wait on a CTA that is not resident
    s_f = a.n_frames > 0 ? static_cast<int>(atomicAdd(&a.psync[0], 1u)) : 0;
  }
  __syncthreads();
  if (a.n_frames == 0) {  // nothing planned: zero totals
    if (tid == 0) plan_totals(a, s_first, 0, 0);
    return;
  }
  const int f = s_f;
#ifdef TG_PLAN_PHASES
  __shared__ long long tg_ph_mark[16];
  TG_PH(0);
#endif
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

  const int nz = a.X * a.Y;
  zone_acc_init(zacc, nz, tid, nt);  // ordered before K3 by the CCL's barriers

  // ---- K2: RoI boxes ---------------------------------------------------------
  const int nr = ccl_frame(a.active + static_cast<size_t>(f) * ncw,
                           a.cells + static_cast<size_t>(f) * cy_n * cx_n, cx_n, cy_n, a.max_rois,
                           cs, warp_tmp, &s_nrois, a.err, f
#ifdef TG_PLAN_PHASES
                           , tg_ph_mark
#endif
                           );
  tg_rect* frois = a.rois + static_cast<size_t>(f) * a.max_rois;
  auto box = [&cs](int r) {
    return tg_rect{cs.bx0[r], cs.by0[r], cs.bx1[r] - cs.bx0[r] + 1, cs.by1[r] - cs.by0[r] + 1};
  };
  for (int r = tid; r < nr; r += nt) frois[r] = box(r);
  if (tid == 0) a.n_rois[f] = nr;

  // ---- K3: partition (Alg. 1) --------------------------------------------
  // straight from the CCL's shared-memory boxes (final after its last barrier)
  partition_accumulate_at(box, nr, a.W, a.H, a.X, a.Y, zacc, a.err, f, nullptr, tid, nt);
  __syncthreads();
  TG_PH(8);
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
  TG_PH(9);

  // ---- K4: stitch plan (Alg. 2 solver) -------------------------------------
  int nfree = 0;
  const int nc = na ? bssf_stitch(adm_w, adm_h, nullptr, na, a.M, a.N, freel, 2 * Z + 2,
                                  souts, &nfree, a.err, f, lane)
                    : 0;
  __syncwarp();
  if (lane == 0) {
    a.n_patches[f] = np;
    a.n_placements[f] = na;
    a.n_canvases[f] = nc < 0 ? 0 : nc;
  }
  TG_PH(10);
  const int ncv = nc < 0 ? 0 : nc;
  look_publish(a, f, s_epoch, static_cast<uint64_t>(np), static_cast<uint64_t>(ncv), lane);
  // Gather jobs (frame-local): placements and free rects grouped by canvas,
  // sorted by x; lane c keeps canvases c, c + 32, ...: (first job, count)
  // for their ranges (a frame has at most Z canvases).
  uint32_t my_rng[Z / 32] = {};  // first job | count << 16
  if (ncv > 0) {
    Job* fj = a.jobs + static_cast<size_t>(f) * a.job_cap;
    uint32_t* fcj = a.canvas_jobs + static_cast<size_t>(f) * nz;
    const int nitems = na + nfree;
    int pos = 0;
    for (int c = 0; c < ncv; ++c) {
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
      if (lane == (c & 31)) my_rng[c >> 5] = static_cast<uint32_t>(pos) | static_cast<uint32_t>(cnt) << 16;
      pos += cnt;
    }
  }
  TG_PH(11);
  // frame-order prefix: global patch ids, canvas numbering
  uint64_t ex_p, ex_c;
  look_back(a, f, s_epoch, static_cast<uint64_t>(np), static_cast<uint64_t>(ncv), &ex_p, &ex_c,
            lane);
  TG_PH(12);
  const uint64_t id0 = s_first + ex_p;
  const long long cb = static_cast<long long>(ex_c);
  for (int j = lane; j < np; j += 32) a.patches[static_cast<size_t>(f) * nz + j].patch_id = id0 + j;
  if (a.desc_head) {  // dense descriptor list: the look-back prefix is the compaction scan
    const int cam = a.desc_cameras ? a.desc_cameras[f / a.desc_fpc] : 0;
    const int fr = a.desc_cameras ? f % a.desc_fpc : f;
    for (int j = lane; j < np; j += 32) {
      const long long k = static_cast<long long>(ex_p) + j;
      if (k >= a.desc_cap) continue;
      tg_descriptor d;
      d.patch = spatch[j];
      d.patch.patch_id = ex_p + j;
      d.camera = cam;
      d.frame = fr;
      d.admitted = (d.patch.rect.w <= a.M && d.patch.rect.h <= a.N) ? 1 : 0;
      d.pad = 0;
      a.desc[k] = d;
    }
  }
  if (lane == 0) {
    a.canvas_base[f] = cb;
    if (f == a.n_frames - 1) plan_totals(a, s_first, ex_p + np, cb + ncv);
  }
#pragma unroll
  for (int h = 0; h < Z / 32; ++h) {
    const int c = lane + 32 * h;
    if (c < ncv && cb + c < a.max_canvases)
      a.ranges[cb + c] = make_uint2(static_cast<uint32_t>(f) * a.job_cap + (my_rng[h] & 0xffffu),
                                    my_rng[h] >> 16);
  }
  tg_placement* fpl = a.placements + static_cast<size_t>(f) * nz;
  for (int k = lane; k < na; k += 32) {
    tg_placement p;
    p.patch_id = id0 + static_cast<uint64_t>(adm_idx[k]);
    p.canvas_index = souts[k].canvas;
    p.position = tg_rect{souts[k].x, souts[k].y, adm_w[k], adm_h[k]};
    p.reserved = 0;
    fpl[k] = p;
  }
#ifdef TG_PLAN_PHASES
  TG_PH(13);
  if (lane == 0) {
    for (int i = 1; i < 14; ++i)
      atomicAdd(&g_plan_phase[i], static_cast<unsigned long long>(tg_ph_mark[i] - tg_ph_mark[i - 1]));
    atomicAdd(&g_plan_phase[0], 1ull);
  }
#endif
  // The last CTA out resets the ticket and moves the epoch on.  Look-back
  // words carry a 16-bit epoch and are never cleared per launch, so every
  // 32768 launches the whole array is zeroed: a surviving word is then less
  // than 32768 launches old and cannot alias the current epoch.
  unsigned last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(&a.psync[1], 1u) == static_cast<uint32_t>(a.n_frames) - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) {
    const uint32_t next = s_epoch + 1;
    if ((next & 0x7fffu) == 0)
      for (int i = lane; i < a.look_cap; i += 32) a.look[i] = 0;
    __syncwarp();
    if (lane == 0) {
      a.psync[0] = 0;
      a.psync[1] = 0;
      __threadfence();
      a.psync[2] = next;
      __threadfence();
    }
  }
}

// ---- drop-in / batched rect-level kernels ---------------------------------
// One block per frame: partition() of host-supplied RoIs.
// Zones are accumulated kMaxZones at a time (any grid, like the reference's
// partition): each chunk's non-empty zones become patches in zone order,
// numbered after the previous chunks'.
__global__ void __launch_bounds__(256) partition_batch_kernel(const PartitionBatchArgs a) {
  __shared__ ZoneAcc zacc;
  __shared__ tg_patch_meta sp[kMaxZones];
  __shared__ int s_base;
  const int f = blockIdx.x, tid = threadIdx.x, nz = a.X * a.Y;
  const tg_frame_spec fs = a.frames[f];
  const int r0 = a.roi_offsets[f], r1 = a.roi_offsets[f + 1];
  const tg_rect* rois = a.rois + r0;
  if (tid == 0) s_base = 0;
  for (int zc = 0; zc < nz; zc += kMaxZones) {
    const int cn = min(kMaxZones, nz - zc);
    zone_acc_init(zacc, cn, tid, blockDim.x);
    __syncthreads();
    for (int i = tid; i < r1 - r0; i += blockDim.x) {
      const tg_rect r = rois[i];
      const int bz = best_zone(r, fs.width, fs.height, a.X, a.Y);
      if (zc == 0) {
        if (a.zone_of) a.zone_of[r0 + i] = bz;
        // with zone_of the caller reports the FIRST bad index itself (the
        // reference throws at the lowest one, partition.hpp:106-108)
        else if (bz < 0) raise_error(a.err, TG_ERR_INVALID_ARGUMENT, kErrRoiOutside, i, f);
      }
      const int zi = bz - zc;
      if (bz < zc || zi >= cn) continue;  // outside the frame, or another chunk's zone
      atomicMin(&zacc.x0[zi], r.x);
      atomicMin(&zacc.y0[zi], r.y);
      atomicMax(&zacc.x1[zi], r.x + r.w);
      atomicMax(&zacc.y1[zi], r.y + r.h);
      atomicAdd(&zacc.cnt[zi], 1);
    }
    __syncthreads();
    if (tid < 32) {
      const int base = s_base;
      const int np = partition_emit(zacc, cn, fs.frame_id, fs.generation_time_us, fs.slo_us,
                                    a.bpp, a.first_ids[f] + static_cast<uint64_t>(base), sp, tid);
      __syncwarp();
      for (int j = tid; j < np; j += 32) a.patches[static_cast<size_t>(f) * nz + base + j] = sp[j];
      __syncwarp();
      if (tid == 0) s_base = base + np;
    }
    __syncthreads();
  }
  if (tid >= 32) return;
  __threadfence_system();  // zone_of / patches may be host-mapped: visible before n_patches
  __syncwarp();
  // n_patches is written last: the blocking drop-in waits on it in mapped
  // host memory instead of synchronizing the stream
  if (tid == 0) a.n_patches[f] = s_base;
}

// One warp per queue; the free set ends in the caller's workspace.  A short
// queue (<= kStitchStage patches) is first staged into shared memory by all
// lanes at once -- the blocking drop-in passes it in mapped host memory,
// where every dependent read would be a PCIe round trip -- and its free set
// is kept in shared memory while it is built (copied out at the end); longer
// queues are read in place and their free set lives in the workspace.  Placements are written in place (no context scratch, so
// stream-ordered batches never share buffers with other calls).

__global__ void __launch_bounds__(128) stitch_batch_kernel(const StitchBatchArgs a) {
  __shared__ int2 s_wh[4][kStitchStage];
  __shared__ unsigned long long s_id[4][kStitchStage];
  __shared__ FreeRect s_fr[4][2 * kStitchStage + 1];
  const int wq = threadIdx.x / 32;
  const int q = blockIdx.x * (blockDim.x / 32) + wq;
  const int lane = threadIdx.x & 31;
  if (q >= a.n_queues) return;
  const int o0 = a.offsets[q], n = a.offsets[q + 1] - o0;
  const tg_patch_meta* qu = a.queue + o0;
  tg_placement* pl = a.placements + o0;
  FreeRect* fl = a.free_ws + 2 * static_cast<size_t>(o0) + q;
  int nfree = 0;
  int nc;
  auto emit = [pl](int i, unsigned long long id, int2 wh, int c, int x, int y) {
    tg_placement p;
    p.patch_id = id;
    p.canvas_index = c;
    p.position = tg_rect{x, y, wh.x, wh.y};
    p.reserved = 0;
    pl[i] = p;
  };
  if (n <= kStitchStage) {
    int2* wh = s_wh[wq];
    unsigned long long* id = s_id[wq];
    for (int i = lane; i < n; i += 32) {
      const tg_patch_meta m = qu[i];
      wh[i] = make_int2(m.rect.w, m.rect.h);
      id[i] = m.patch_id;
    }
    __syncwarp();
    // the free set too: every placement scans and rewrites it
    FreeRect* sfl = s_fr[wq];
    nc = bssf_stitch_q([wh](int i) { return wh[i]; }, [id](int i) { return id[i]; },
                       [wh, id, emit](int i, int c, int x, int y) { emit(i, id[i], wh[i], c, x, y); },
                       n, a.M, a.N, sfl, 2 * n + 1, &nfree, a.err, q, lane);
    __syncwarp();
    for (int i = lane; i < nfree; i += 32) fl[i] = sfl[i];
  } else {
    nc = bssf_stitch_q(
        [qu](int i) { return make_int2(qu[i].rect.w, qu[i].rect.h); },
        [qu](int i) { return qu[i].patch_id; },
        [qu, emit](int i, int c, int x, int y) {
          emit(i, qu[i].patch_id, make_int2(qu[i].rect.w, qu[i].rect.h), c, x, y);
        },
        n, a.M, a.N, fl, 2 * n + 1, &nfree, a.err, q, lane);
  }
  // n_canvases is written last: the blocking drop-in waits on it in mapped
  // host memory instead of synchronizing the stream
  __threadfence_system();
  __syncwarp();
  if (lane == 0) {
    if (a.n_free) a.n_free[q] = nfree;
    __threadfence_system();
    a.n_canvases[q] = nc;
  }
}

// ---- launchers --------------------------------------------------------------
size_t plan_smem_bytes(int cells_x, int cells_y, int max_rois, int zones) {
  const int aw = ceil_div(cells_x, 32);
  const size_t ncw = static_cast<size_t>(cells_y) * aw;
  const size_t ccl = ncw * 4 * 2 + (ncw + 1) * 4 + static_cast<size_t>(max_rois) * 16 +
                     ncw * kHeadsPerWord * 2 + 16;
  const size_t tail = zones <= kMaxZones ? sizeof(PlanTail<kMaxZones>)
                                         : sizeof(PlanTail<kMaxPlanZones>);
  return ccl > tail ? ccl : tail;
}

template <int Z>
static cudaError_t launch_plan_t(const PlanArgs& a, size_t smem, cudaStream_t stream) {
  static SmemOptIn opt_in;
  cudaError_t e = opt_in.ensure(plan_kernel<Z>, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  plan_kernel<Z><<<a.n_frames > 0 ? a.n_frames : 1, kPlanThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream) {
  if (a.n_frames < 0) return cudaErrorInvalidValue;
  const int nz = a.X * a.Y;
  if (nz > kMaxPlanZones) return cudaErrorInvalidValue;
  const size_t smem = plan_smem_bytes(a.cells_x, a.cells_y, a.max_rois, nz);
  return nz <= kMaxZones ? launch_plan_t<kMaxZones>(a, smem, stream)
                         : launch_plan_t<kMaxPlanZones>(a, smem, stream);
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

#ifdef TG_PLAN_PHASES
// Diagnostics build only: phase cycle sums of thread 0 over all frame CTAs
// since the last call (out[0] = CTA count); resets them.
extern "C" int tg_debug_plan_phases(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, tg::g_plan_phase, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {};
  return static_cast<int>(cudaMemcpyToSymbol(tg::g_plan_phase, z, sizeof(z)));
}
#endif
