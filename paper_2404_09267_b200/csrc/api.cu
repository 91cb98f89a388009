// api.cu -- the C ABI (include/tangram_gpu.h) over the sm_100a kernels.
//
// Host-side responsibilities only: argument validation with the reference's
// error texts, device memory for the per-frame result slots, stream-ordered
// launches, CUDA-graph capture, and turning latched device errors back into
// status codes + messages.  No pixel or rect work happens on the host, and
// there is no CPU fallback: every compute entry point returns
// TG_ERR_NO_DEVICE when no CUDA device is usable.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "rect_core.cuh"
#include "tangram_gpu.h"

using namespace tg;

namespace {

thread_local std::string g_err;

tg_status fail(tg_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

tg_status cuda_fail(cudaError_t e, const char* what) {
  return fail(TG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define TG_CUDA(expr)                                   \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

}  // namespace

struct tg_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  DevError* d_err = nullptr;
  // grow-only scratch for the blocking drop-in calls
  void* d_scratch = nullptr;
  size_t scratch_bytes = 0;
  // pinned, device-mapped staging of the blocking drop-in calls: the host
  // writes inputs the kernel reads in place and reads outputs the kernel
  // wrote (zero copy), so a call is one launch + one synchronization
  uint8_t* h_stage = nullptr;
  uint8_t* d_stage = nullptr;
  size_t stage_bytes = 0;
  // stream-ordered staging for explicit gather plans (tg_stitch_gather,
  // tg_batcher_gather)
  Job* g_jobs = nullptr;
  uint2* g_ranges = nullptr;
  int32_t* g_units = nullptr;
  int32_t g_units_h[3] = {0, 0, 0};
  size_t g_job_cap = 0, g_range_cap = 0;
  int32_t gather_grid = 0;  // TG_OPT_GATHER_GRID (0: SMs x the occupancy limit)
  int32_t gather_band = 0;  // TG_OPT_GATHER_BAND (0: gather_band())
};

struct tg_pipeline {
  tg_ctx* ctx = nullptr;
  tg_pipeline_params p{};
  int zones = 0, cells_x = 0, cells_y = 0, act_words = 0, mask_words = 0, job_cap = 0, nbands = 0;
  uint32_t *raw = nullptr, *cells = nullptr, *active = nullptr, *mask = nullptr;
  uint32_t* mask_sync = nullptr;  // fused K1/K1b launch: item counters + task queue
  int32_t *n_rois = nullptr, *n_patches = nullptr, *n_placements = nullptr, *n_canvases = nullptr;
  tg_rect* rois = nullptr;
  tg_patch_meta* patches = nullptr;
  uint8_t* admitted = nullptr;
  tg_placement* placements = nullptr;
  int64_t* canvas_base = nullptr;
  Job* jobs = nullptr;
  uint32_t* canvas_jobs = nullptr;
  uint2* ranges = nullptr;
  int32_t* gather_units = nullptr;
  uint64_t* id_state = nullptr;
  uint64_t* look = nullptr;   // [F] plan look-back words
  uint32_t* psync = nullptr;  // [3] plan frame ticket, finished CTAs, epoch
  int last_frames = 0;
  tg_pipeline_stats stats{};
  // optional dense descriptor output (tg_pipeline_set_descriptor_output)
  tg_descriptor_header* desc_head = nullptr;
  int64_t desc_cap = 0;
  const int32_t* desc_cameras = nullptr;
  int32_t desc_fpc = 1;
};

struct tg_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

namespace {

tg_status use_device(tg_ctx* ctx) {
  if (!ctx) return fail(TG_ERR_INVALID_ARGUMENT, "null context");
  TG_CUDA(cudaSetDevice(ctx->device));
  return TG_OK;
}

cudaStream_t pick(tg_ctx* ctx, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
}

tg_status device_error_status(const DevError& e);

// Reads and clears the device error latch.
tg_status check_device_error(tg_ctx* ctx) {
  DevError e;
  TG_CUDA(cudaMemcpy(&e, ctx->d_err, sizeof(e), cudaMemcpyDeviceToHost));
  if (e.code == 0) return TG_OK;
  TG_CUDA(cudaMemset(ctx->d_err, 0, sizeof(DevError)));
  TG_CUDA(cudaDeviceSynchronize());  // the legacy-stream reset precedes later launches
  return device_error_status(e);
}

tg_status device_error_status(const DevError& e) {
  switch (e.kind) {
    case kErrRoiOutside:  // partition.hpp:106-108
      return fail(static_cast<tg_status>(e.code), "roi outside frame (roi index %lld)", e.a);
    case kErrPatchOversize:  // stitch.hpp:114-118
      return fail(static_cast<tg_status>(e.code), "patch exceeds canvas (patch %llu, %lldx%lld)",
                  static_cast<unsigned long long>(e.a), e.b, e.c);
    case kErrRoiCapacity:
      return fail(static_cast<tg_status>(e.code),
                  "roi capacity exceeded (frame %lld: %lld components > %lld slots)", e.a, e.b, e.c);
    case kErrCanvasCapacity:
      return fail(static_cast<tg_status>(e.code), "canvas capacity exceeded (%lld canvases > %lld)",
                  e.a, e.b);
    case kErrFreeCapacity:
      return fail(static_cast<tg_status>(e.code), "free rect capacity exceeded (queue %lld)", e.a);
    case kErrDescCapacity:
      return fail(static_cast<tg_status>(e.code),
                  "descriptor capacity exceeded (%lld patches > %lld records)", e.a, e.b);
    default:
      return fail(static_cast<tg_status>(e.code), "device error kind %d", e.kind);
  }
}

tg_status scratch(tg_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->d_scratch) TG_CUDA(cudaFree(ctx->d_scratch));
    ctx->d_scratch = nullptr;
    ctx->scratch_bytes = 0;
    const size_t want = std::max<size_t>(bytes, 1 << 20);
    TG_CUDA(cudaMalloc(&ctx->d_scratch, want));
    ctx->scratch_bytes = want;
  }
  *out = ctx->d_scratch;
  return TG_OK;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Waits until a kernel of the blocking drop-in path has written its result
// flag (its last store, after a system-scope fence) into mapped host memory:
// a spin on host memory instead of a stream synchronization.  After 20 ms it
// synchronizes the stream instead, which also reports a failed launch.
tg_status await_flag(tg_ctx* ctx, const int32_t* flag, int32_t sentinel) {
  const volatile int32_t* f = flag;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t it = 1; *f == sentinel; ++it) {
    if ((it & 1023u) == 0 &&
        std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(20)) {
      TG_CUDA(cudaStreamSynchronize(ctx->stream));
      if (*f == sentinel) return fail(TG_ERR_CUDA, "device call finished without a result");
      break;
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return TG_OK;
}

tg_status stage(tg_ctx* ctx, size_t bytes, uint8_t** h, uint8_t** d) {
  if (bytes > ctx->stage_bytes) {
    if (ctx->h_stage) TG_CUDA(cudaFreeHost(ctx->h_stage));
    ctx->h_stage = ctx->d_stage = nullptr;
    ctx->stage_bytes = 0;
    const size_t want = std::max<size_t>(align_up(bytes, 4096), 64 << 10);
    TG_CUDA(cudaHostAlloc(&ctx->h_stage, want, cudaHostAllocMapped));
    TG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_stage), ctx->h_stage, 0));
    ctx->stage_bytes = want;
  }
  *h = ctx->h_stage;
  *d = ctx->d_stage;
  return TG_OK;
}

// Lays out several arrays in one scratch allocation.
struct Carver {
  size_t off = 0;
  template <class T>
  size_t take(size_t count) {
    off = align_up(off, 256);
    const size_t at = off;
    off += count * sizeof(T);
    return at;
  }
};

// partition.hpp:70-73.  `device_limit`: the fused per-frame planner keeps a
// frame's zones in shared memory (kMaxZones); the drop-in partition takes
// any grid, like the reference.
tg_status zone_grid_check(int width, int height, tg_partition_config cfg, bool device_limit) {
  if (cfg.zones_x < 1 || cfg.zones_y < 1 || cfg.zones_x > width || cfg.zones_y > height)
    return fail(TG_ERR_INVALID_ARGUMENT, "zone grid finer than frame");
  if (device_limit && cfg.zones_x * cfg.zones_y > kMaxPlanZones)
    return fail(TG_ERR_INVALID_ARGUMENT, "zone grid exceeds the pipeline limit (%d zones)",
                kMaxPlanZones);
  if (static_cast<long long>(cfg.zones_x) * cfg.zones_y > (1 << 24))
    return fail(TG_ERR_INVALID_ARGUMENT, "zone grid too large");
  return TG_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int tg_abi_version(void) { return TG_ABI_VERSION; }

// ---- internal hooks for batcher.cu / comm.cu (not part of the public header) --
void tg_internal_set_error(const char* msg) { g_err = msg; }
int tg_internal_ctx_device(tg_ctx* ctx) { return ctx ? ctx->device : -1; }

// Uploads an explicit gather plan (host Job[] + per-canvas ranges) on the
// stream and launches K5 over it.  Pageable host sources: cudaMemcpyAsync
// returns once they are consumed, so callers may free them immediately.
tg_status tg_internal_run_gather(tg_ctx* ctx, const void* jobs, int32_t n_jobs, const void* ranges,
                                 int32_t n_canvases, tg_canvas_spec spec,
                                 const uint8_t* const* d_frames, int32_t pitch, uint8_t* d_out,
                                 void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if (n_canvases == 0) return TG_OK;
  if (!d_out || !d_frames) return fail(TG_ERR_INVALID_ARGUMENT, "null frame table or canvas buffer");
  cudaStream_t st = pick(ctx, stream);
  if (static_cast<size_t>(n_jobs) > ctx->g_job_cap) {
    TG_CUDA(cudaStreamSynchronize(st));
    if (ctx->g_jobs) TG_CUDA(cudaFree(ctx->g_jobs));
    ctx->g_job_cap = std::max<size_t>(n_jobs, 4096);
    TG_CUDA(cudaMalloc(&ctx->g_jobs, ctx->g_job_cap * sizeof(Job)));
  }
  if (static_cast<size_t>(n_canvases) > ctx->g_range_cap) {
    TG_CUDA(cudaStreamSynchronize(st));
    if (ctx->g_ranges) TG_CUDA(cudaFree(ctx->g_ranges));
    ctx->g_range_cap = std::max<size_t>(n_canvases, 1024);
    TG_CUDA(cudaMalloc(&ctx->g_ranges, ctx->g_range_cap * sizeof(uint2)));
  }
  if (!ctx->g_units) TG_CUDA(cudaMalloc(&ctx->g_units, 3 * sizeof(int32_t)));
  const int band =
      ctx->gather_band > 0 ? ctx->gather_band : gather_band(n_canvases, spec.height, ctx->sms);
  const int nbands = gather_bands(spec.height, band);
  ctx->g_units_h[0] = n_canvases * nbands;
  ctx->g_units_h[1] = 0;  // K5's unit claim counter
  ctx->g_units_h[2] = 0;  // K5's finished-CTA counter
  if (n_jobs > 0)
    TG_CUDA(cudaMemcpyAsync(ctx->g_jobs, jobs, sizeof(Job) * n_jobs, cudaMemcpyHostToDevice, st));
  TG_CUDA(cudaMemcpyAsync(ctx->g_ranges, ranges, sizeof(uint2) * n_canvases,
                          cudaMemcpyHostToDevice, st));
  TG_CUDA(cudaMemcpyAsync(ctx->g_units, ctx->g_units_h, 3 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GatherArgs g;
  g.frames = d_frames;
  g.pitch = pitch;
  g.M = spec.width;
  g.N = spec.height;
  g.nbands = nbands;
  g.band = band;
  g.jobs = ctx->g_jobs;
  g.ranges = ctx->g_ranges;
  g.units = ctx->g_units;
  g.out = d_out;
  TG_CUDA(launch_gather(g, ctx->sms, ctx->gather_grid, st));
  return TG_OK;
}

const char* tg_last_error(void) { return g_err.c_str(); }

tg_status tg_device_count(int32_t* count) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  *count = n;
  return TG_OK;
}

tg_status tg_ctx_create(int32_t device, tg_ctx** out) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(TG_ERR_NO_DEVICE, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(TG_ERR_INVALID_ARGUMENT, "bad device %d", device);
  TG_CUDA(cudaSetDevice(device));
  tg_ctx* c = new tg_ctx();
  c->device = device;
  TG_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
  TG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  TG_CUDA(cudaMalloc(&c->d_err, sizeof(DevError)));
  TG_CUDA(cudaMemset(c->d_err, 0, sizeof(DevError)));
  TG_CUDA(cudaDeviceSynchronize());  // before any non-blocking stream's kernel can latch
  *out = c;
  return TG_OK;
}

void tg_ctx_destroy(tg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->g_jobs) cudaFree(ctx->g_jobs);
  if (ctx->g_ranges) cudaFree(ctx->g_ranges);
  if (ctx->g_units) cudaFree(ctx->g_units);
  cudaFree(ctx->d_err);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void* tg_ctx_stream(tg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

tg_status tg_ctx_synchronize(tg_ctx* ctx) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaDeviceSynchronize());
  return check_device_error(ctx);
}

tg_status tg_ctx_set_option(tg_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return fail(TG_ERR_INVALID_ARGUMENT, "null context");
  switch (option) {
    case TG_OPT_GATHER_GRID:
      if (value < 0 || value > (1 << 20)) return fail(TG_ERR_INVALID_ARGUMENT, "gather grid out of range");
      ctx->gather_grid = static_cast<int32_t>(value);
      return TG_OK;
    case TG_OPT_GATHER_BAND:
      if (value < 0 || value > (1 << 16)) return fail(TG_ERR_INVALID_ARGUMENT, "gather band out of range");
      ctx->gather_band = static_cast<int32_t>(value);
      return TG_OK;
    default:
      return fail(TG_ERR_INVALID_ARGUMENT, "unknown context option %d", option);
  }
}

tg_status tg_device_sm_count(tg_ctx* ctx, int32_t* sms) {
  if (!ctx) return fail(TG_ERR_INVALID_ARGUMENT, "null context");
  *sms = ctx->sms;
  return TG_OK;
}

// ---- memory / streams / events ----------------------------------------------
tg_status tg_malloc_device(tg_ctx* ctx, size_t bytes, void** d_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaMalloc(d_ptr, bytes));
  return TG_OK;
}

tg_status tg_free_device(tg_ctx* ctx, void* d_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaFree(d_ptr));
  return TG_OK;
}

tg_status tg_malloc_host(tg_ctx* ctx, size_t bytes, void** h_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaMallocHost(h_ptr, bytes));
  return TG_OK;
}

tg_status tg_ipc_export(tg_ctx* ctx, void* d_ptr, tg_ipc_handle* out) {
  tg_status s = use_device(ctx);
  if (s) return s;
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(tg_ipc_handle), "ipc handle size");
  cudaIpcMemHandle_t h;
  TG_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
  memset(out, 0, sizeof(*out));
  memcpy(out->bytes, &h, sizeof(h));
  return TG_OK;
}

tg_status tg_ipc_import(tg_ctx* ctx, const tg_ipc_handle* handle, void** d_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle->bytes, sizeof(h));
  TG_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TG_OK;
}

tg_status tg_ipc_close(tg_ctx* ctx, void* d_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return TG_OK;
}

tg_status tg_free_host(tg_ctx* ctx, void* h_ptr) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaFreeHost(h_ptr));
  return TG_OK;
}

tg_status tg_memcpy_async(tg_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind,
                          void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost
                                       : cudaMemcpyDeviceToDevice;
  TG_CUDA(cudaMemcpyAsync(dst, src, bytes, k, pick(ctx, stream)));
  return TG_OK;
}

tg_status tg_memset_async(tg_ctx* ctx, void* d_ptr, int32_t value, size_t bytes, void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaMemsetAsync(d_ptr, value, bytes, pick(ctx, stream)));
  return TG_OK;
}

tg_status tg_stream_create(tg_ctx* ctx, void** stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  cudaStream_t st;
  TG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  *stream = st;
  return TG_OK;
}

tg_status tg_stream_create_priority(tg_ctx* ctx, int32_t high, void** stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  int least = 0, greatest = 0;
  TG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t st;
  TG_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, high ? greatest : least));
  *stream = st;
  return TG_OK;
}

tg_status tg_stream_destroy(tg_ctx* ctx, void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  return TG_OK;
}

tg_status tg_stream_synchronize(tg_ctx* ctx, void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaStreamSynchronize(pick(ctx, stream)));
  return check_device_error(ctx);
}

tg_status tg_event_create(tg_ctx* ctx, void** event) {
  tg_status s = use_device(ctx);
  if (s) return s;
  cudaEvent_t ev;
  TG_CUDA(cudaEventCreate(&ev));
  *event = ev;
  return TG_OK;
}

tg_status tg_event_destroy(tg_ctx* ctx, void* event) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
  return TG_OK;
}

tg_status tg_event_record(tg_ctx* ctx, void* event, void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), pick(ctx, stream)));
  return TG_OK;
}

tg_status tg_event_elapsed_ms(tg_ctx* ctx, void* start, void* stop, float* ms) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(stop)));
  TG_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                               static_cast<cudaEvent_t>(stop)));
  return TG_OK;
}

tg_status tg_event_synchronize(tg_ctx* ctx, void* event) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(event)));
  return TG_OK;
}

tg_status tg_stream_wait_event(tg_ctx* ctx, void* stream, void* event) {
  tg_status s = use_device(ctx);
  if (s) return s;
  TG_CUDA(cudaStreamWaitEvent(pick(ctx, stream), static_cast<cudaEvent_t>(event), 0));
  return TG_OK;
}

// ---- drop-in rect-level API -----------------------------------------------------
tg_status tg_make_zones(const tg_frame_spec* frame, tg_partition_config cfg, tg_rect* zones,
                        int32_t zones_cap) {
  // partition.hpp:69-88 (pure host arithmetic).
  if (cfg.zones_x < 1 || cfg.zones_y < 1 || cfg.zones_x > frame->width ||
      cfg.zones_y > frame->height)
    return fail(TG_ERR_INVALID_ARGUMENT, "zone grid finer than frame");
  if (static_cast<long long>(cfg.zones_x) * cfg.zones_y > zones_cap)
    return fail(TG_ERR_CAPACITY, "zones buffer too small");
  const int zw = frame->width / cfg.zones_x, zh = frame->height / cfg.zones_y;
  int k = 0;
  for (int row = 0; row < cfg.zones_y; ++row) {
    const int y = row * zh;
    const int h = (row == cfg.zones_y - 1) ? frame->height - y : zh;
    for (int col = 0; col < cfg.zones_x; ++col) {
      const int x = col * zw;
      zones[k++] = tg_rect{x, y, (col == cfg.zones_x - 1) ? frame->width - x : zw, h};
    }
  }
  return TG_OK;
}

}  // extern "C"

namespace {
// assign_rois over an explicit zone list (partition.hpp:93-112).
__global__ void assign_kernel(const tg_rect* rois, int n, const tg_rect* zones, int nz,
                              int32_t* zone_of) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long best = 0;
  int bz = -1;
  for (int z = 0; z < nz; ++z) {
    const long long s = tg::overlap_area(rois[i], zones[z]);
    if (s > best) {
      best = s;
      bz = z;
    }
  }
  zone_of[i] = bz;
}
}  // namespace

extern "C" {

tg_status tg_assign_rois(tg_ctx* ctx, const tg_rect* rois, int32_t n_rois, const tg_rect* zones,
                         int32_t n_zones, int32_t* zone_of) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if (n_rois <= 0) return TG_OK;
  Carver cv;
  const size_t o_r = cv.take<tg_rect>(n_rois), o_z = cv.take<tg_rect>(std::max(1, n_zones)),
               o_o = cv.take<int32_t>(n_rois);
  uint8_t *h, *d;
  if ((s = stage(ctx, cv.off, &h, &d))) return s;
  memcpy(h + o_r, rois, sizeof(tg_rect) * n_rois);
  if (n_zones > 0) memcpy(h + o_z, zones, sizeof(tg_rect) * n_zones);
  cudaStream_t st = ctx->stream;
  assign_kernel<<<(n_rois + 127) / 128, 128, 0, st>>>(
      reinterpret_cast<tg_rect*>(d + o_r), n_rois, reinterpret_cast<tg_rect*>(d + o_z), n_zones,
      reinterpret_cast<int32_t*>(d + o_o));
  TG_CUDA(cudaGetLastError());
  TG_CUDA(cudaStreamSynchronize(st));
  memcpy(zone_of, h + o_o, sizeof(int32_t) * n_rois);
  for (int i = 0; i < n_rois; ++i)
    if (zone_of[i] < 0) return fail(TG_ERR_INVALID_ARGUMENT, "roi outside frame (roi index %d)", i);
  return TG_OK;
}

tg_status tg_partition(tg_ctx* ctx, const tg_frame_spec* frame, tg_partition_config cfg,
                       const tg_rect* rois, int32_t n_rois, double bytes_per_pixel,
                       uint64_t first_patch_id, tg_patch_meta* patches, int32_t patches_cap,
                       int32_t* n_patches) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if ((s = zone_grid_check(frame->width, frame->height, cfg, false))) return s;
  const int nz = cfg.zones_x * cfg.zones_y;
  Carver cv;
  const size_t o_f = cv.take<tg_frame_spec>(1), o_off = cv.take<int32_t>(2),
               o_r = cv.take<tg_rect>(std::max(1, n_rois)), o_id = cv.take<uint64_t>(1),
               o_p = cv.take<tg_patch_meta>(nz), o_n = cv.take<int32_t>(1),
               o_z = cv.take<int32_t>(std::max(1, n_rois));
  uint8_t *h, *d;
  if ((s = stage(ctx, cv.off, &h, &d))) return s;
  const int32_t offs[2] = {0, n_rois};
  memcpy(h + o_f, frame, sizeof(tg_frame_spec));
  memcpy(h + o_off, offs, sizeof(offs));
  if (n_rois > 0) memcpy(h + o_r, rois, sizeof(tg_rect) * n_rois);
  memcpy(h + o_id, &first_patch_id, 8);
  const int32_t pending = -1;
  memcpy(h + o_n, &pending, 4);
  cudaStream_t st = ctx->stream;
  PartitionBatchArgs a;
  a.n_frames = 1;
  a.X = cfg.zones_x;
  a.Y = cfg.zones_y;
  a.bpp = bytes_per_pixel;
  a.frames = reinterpret_cast<tg_frame_spec*>(d + o_f);
  a.roi_offsets = reinterpret_cast<int32_t*>(d + o_off);
  a.rois = reinterpret_cast<tg_rect*>(d + o_r);
  a.first_ids = reinterpret_cast<uint64_t*>(d + o_id);
  a.patches = reinterpret_cast<tg_patch_meta*>(d + o_p);
  a.n_patches = reinterpret_cast<int32_t*>(d + o_n);
  a.zone_of = reinterpret_cast<int32_t*>(d + o_z);
  a.err = ctx->d_err;
  TG_CUDA(launch_partition_batch(a, st));
  // with zone_of the kernel latches no error: an RoI outside the frame shows
  // as zone -1, reported below at the lowest index like the reference
  if ((s = await_flag(ctx, reinterpret_cast<const int32_t*>(h + o_n), pending))) return s;
  const int32_t* zone_of = reinterpret_cast<const int32_t*>(h + o_z);
  for (int i = 0; i < n_rois; ++i)  // the reference throws at the first bad index
    if (zone_of[i] < 0) return fail(TG_ERR_INVALID_ARGUMENT, "roi outside frame (roi index %d)", i);
  int32_t np = 0;
  memcpy(&np, h + o_n, 4);
  if (np > patches_cap) return fail(TG_ERR_CAPACITY, "patches buffer too small (%d patches)", np);
  if (np > 0) memcpy(patches, h + o_p, sizeof(tg_patch_meta) * np);
  *n_patches = np;
  return TG_OK;
}

tg_status tg_stitch_batch(tg_ctx* ctx, int32_t n_queues, int32_t total_patches,
                          const int32_t* d_queue_offsets, const tg_patch_meta* d_queue,
                          tg_canvas_spec spec, tg_placement* d_placements,
                          int32_t* d_n_canvases, tg_free_rect* d_free_ws, int32_t* d_n_free,
                          void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if (spec.width < 1 || spec.height < 1 || spec.width > 65535 || spec.height > 65535)
    return fail(TG_ERR_INVALID_ARGUMENT, "canvas dimensions must be in [1, 65535]");
  if (n_queues <= 0) return TG_OK;
  StitchBatchArgs a;
  a.n_queues = n_queues;
  a.M = spec.width;
  a.N = spec.height;
  a.offsets = d_queue_offsets;
  a.queue = d_queue;
  a.placements = d_placements;
  a.n_canvases = d_n_canvases;
  a.free_ws = reinterpret_cast<FreeRect*>(d_free_ws);
  a.n_free = d_n_free;
  a.err = ctx->d_err;
  TG_CUDA(launch_stitch_batch(a, pick(ctx, stream)));
  return TG_OK;
}

tg_status tg_stitch_all(tg_ctx* ctx, const tg_patch_meta* queue, int32_t n, tg_canvas_spec spec,
                        tg_placement* placements, int32_t* n_canvases, tg_free_rect* free_rects,
                        int32_t free_cap, int32_t* n_free) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if (spec.width < 1 || spec.height < 1 || spec.width > 65535 || spec.height > 65535)
    return fail(TG_ERR_INVALID_ARGUMENT, "canvas dimensions must be in [1, 65535]");
  if (n <= 0) {
    *n_canvases = 0;
    if (n_free) *n_free = 0;
    return TG_OK;
  }
  // queue in, placements, counts and the final free list out through the
  // mapped staging; the kernel builds a short queue's free list in shared
  // memory (a long one's in device scratch, copied back after a sync)
  const bool staged = n <= kStitchStage;
  const size_t nfr = 2 * static_cast<size_t>(n) + 1;
  Carver cv;
  const size_t o_q = cv.take<tg_patch_meta>(n), o_off = cv.take<int32_t>(2),
               o_pl = cv.take<tg_placement>(n), o_nc = cv.take<int32_t>(1),
               o_nf = cv.take<int32_t>(1), o_fh = cv.take<tg_free_rect>(nfr);
  uint8_t *h, *d;
  if ((s = stage(ctx, cv.off, &h, &d))) return s;
  void* fr_dev = d + o_fh;
  if (!staged && (s = scratch(ctx, nfr * sizeof(tg_free_rect), &fr_dev))) return s;
  const int32_t offs[2] = {0, n};
  const int32_t pending = INT_MIN;
  memcpy(h + o_q, queue, sizeof(tg_patch_meta) * n);
  memcpy(h + o_off, offs, sizeof(offs));
  memcpy(h + o_nc, &pending, 4);
  cudaStream_t st = ctx->stream;
  StitchBatchArgs a;
  a.n_queues = 1;
  a.M = spec.width;
  a.N = spec.height;
  a.offsets = reinterpret_cast<int32_t*>(d + o_off);
  a.queue = reinterpret_cast<tg_patch_meta*>(d + o_q);
  a.placements = reinterpret_cast<tg_placement*>(d + o_pl);
  a.n_canvases = reinterpret_cast<int32_t*>(d + o_nc);
  a.free_ws = static_cast<FreeRect*>(fr_dev);
  a.n_free = reinterpret_cast<int32_t*>(d + o_nf);
  a.err = ctx->d_err;
  TG_CUDA(launch_stitch_batch(a, st));
  if (staged) {
    if ((s = await_flag(ctx, reinterpret_cast<const int32_t*>(h + o_nc), pending))) return s;
  } else {
    if (free_rects)
      TG_CUDA(cudaMemcpyAsync(h + o_fh, fr_dev, nfr * sizeof(tg_free_rect), cudaMemcpyDeviceToHost, st));
    TG_CUDA(cudaStreamSynchronize(st));
  }
  int32_t nc = 0, nf = 0;
  memcpy(&nc, h + o_nc, 4);
  if (nc < 0) {  // the kernel latched an error (oversize patch / capacity)
    if ((s = check_device_error(ctx))) return s;
    return fail(TG_ERR_CUDA, "stitch failed without a latched error");
  }
  memcpy(&nf, h + o_nf, 4);
  memcpy(placements, h + o_pl, sizeof(tg_placement) * n);
  *n_canvases = nc;
  if (n_free) *n_free = nf;
  if (free_rects) {
    if (nf > free_cap) return fail(TG_ERR_CAPACITY, "free rect buffer too small (%d rects)", nf);
    tg_free_rect* fr = reinterpret_cast<tg_free_rect*>(h + o_fh);
    std::sort(fr, fr + nf, [](const tg_free_rect& x, const tg_free_rect& y) {
      return x.canvas_index != y.canvas_index ? x.canvas_index < y.canvas_index : x.seq < y.seq;
    });
    std::copy(fr, fr + nf, free_rects);
  }
  return TG_OK;
}

// ---- the hot path ------------------------------------------------------------------
tg_status tg_pipeline_params_default(int32_t width, int32_t height, tg_pipeline_params* out) {
  tg_pipeline_params p{};
  p.width = width;
  p.height = height;
  p.pitch = 3 * width;
  p.threshold = 25;
  p.dilate_radius = 2;
  p.partition = tg_partition_config{4, 4};     // partition.hpp:50-51
  p.canvas = tg_canvas_spec{1024, 1024, 1.0};  // stitch.hpp:33-35
  p.bytes_per_pixel = 1.5;                     // trace.hpp:238
  p.slo_us = 1000000;
  p.max_frames = 300;
  p.max_rois_per_frame = 1024;
  p.max_canvases = 0;
  p.keep_mask = 0;
  *out = p;
  return TG_OK;
}

void tg_pipeline_destroy(tg_pipeline* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  void* bufs[] = {p->raw, p->mask_sync, p->cells, p->mask, p->n_rois, p->n_patches, p->n_placements,
                  p->n_canvases, p->rois, p->patches, p->admitted, p->placements,
                  p->canvas_base, p->jobs, p->canvas_jobs, p->ranges, p->gather_units,
                  p->id_state, p->look, p->psync};
  for (void* b : bufs)
    if (b) cudaFree(b);
  delete p;
}

tg_status tg_pipeline_create(tg_ctx* ctx, const tg_pipeline_params* params, tg_pipeline** out) {
  *out = nullptr;
  tg_status s = use_device(ctx);
  if (s) return s;
  const tg_pipeline_params& q = *params;
  if (q.width < 16 || q.height < 1 || q.width % 16 != 0 || q.width > 32 * 256)
    return fail(TG_ERR_INVALID_ARGUMENT, "frame width must be a multiple of 16 in [16, 8192]");
  if (q.height > 65535) return fail(TG_ERR_INVALID_ARGUMENT, "frame height must be <= 65535");
  if (q.pitch < 3 * q.width || q.pitch % 16 != 0)
    return fail(TG_ERR_INVALID_ARGUMENT, "pitch must be >= 3*width and a multiple of 16");
  if (q.threshold < 0 || q.threshold > 255)
    return fail(TG_ERR_INVALID_ARGUMENT, "threshold must be in [0, 255]");
  if (q.dilate_radius < 0 || q.dilate_radius > kMaxRadius)
    return fail(TG_ERR_INVALID_ARGUMENT, "dilate radius must be in [0, %d]", kMaxRadius);
  if ((s = zone_grid_check(q.width, q.height, q.partition, true))) return s;
  if (q.canvas.width < 1 || q.canvas.height < 1 || q.canvas.width > 65535 ||
      q.canvas.height > 65535)
    return fail(TG_ERR_INVALID_ARGUMENT, "canvas dimensions must be in [1, 65535]");
  if (q.max_frames < 1 || q.max_rois_per_frame < 1 || q.max_canvases < 0)
    return fail(TG_ERR_INVALID_ARGUMENT, "capacities must be positive");
  const int cx = q.width / kCell, cy = ceil_div(q.height, kCell);
  if (static_cast<long long>(cx) * cy > 65535 ||
      static_cast<long long>(ceil_div(cx, 32)) * cy * 16 > 65536)  // 16-bit CCL run slots
    return fail(TG_ERR_INVALID_ARGUMENT, "frame has more than 65535 %dx%d cells", kCell, kCell);
  if (plan_smem_bytes(cx, cy, q.max_rois_per_frame,
                      q.partition.zones_x * q.partition.zones_y) > 200 * 1024)
    return fail(TG_ERR_INVALID_ARGUMENT, "max_rois_per_frame too large for this frame size");
  // patch and canvas prefixes travel in 23-bit look-back fields
  if (static_cast<long long>(q.max_frames) * q.partition.zones_x * q.partition.zones_y >= (1 << 23))
    return fail(TG_ERR_INVALID_ARGUMENT, "max_frames x zones must be below 2^23");
  tg_pipeline* p = new tg_pipeline();
  p->ctx = ctx;
  p->p = q;
  p->zones = q.partition.zones_x * q.partition.zones_y;
  p->cells_x = cx;
  p->cells_y = cy;
  p->act_words = ceil_div(cx, 32);
  p->mask_words = ceil_div(q.width, 32);
  p->job_cap = 3 * p->zones;
  p->nbands = gather_bands(q.canvas.height, kGatherDefaultBand);
  const size_t F = q.max_frames, Z = p->zones;
  auto alloc = [&](auto** ptr, size_t count) -> cudaError_t {
    return cudaMalloc(reinterpret_cast<void**>(ptr), std::max<size_t>(1, count) * sizeof(**ptr));
  };
  cudaError_t e = cudaSuccess;
  // F raw frames + one zero frame (K1b's rows for columns outside the frame)
  // ... then, split launches, the sparse bitmap's per-row word flags
  // (kernels.cuh: raw_flag_words)
  if (!e) e = alloc(&p->raw, (F + 1) * q.height * p->mask_words +
                                 F * q.height * raw_flag_words(q.width));
  if (!e) e = cudaMemset(p->raw + F * q.height * p->mask_words, 0,
                         q.height * p->mask_words * sizeof(uint32_t));
  // K1 counters followed by the activity bits (p->active): one memset per launch
  const size_t sync_words = mask_sync_words(q.height, ctx->sms);
  if (!e) e = alloc(&p->mask_sync, sync_words + F * cy * p->act_words);
  if (!e) p->active = p->mask_sync + sync_words;
  if (!e) e = alloc(&p->cells, F * cx * cy);
  if (!e && q.keep_mask) e = alloc(&p->mask, F * q.height * p->mask_words);
  if (!e) e = alloc(&p->n_rois, F);
  if (!e) e = alloc(&p->rois, F * q.max_rois_per_frame);
  if (!e) e = alloc(&p->n_patches, F);
  if (!e) e = alloc(&p->patches, F * Z);
  if (!e) e = alloc(&p->admitted, F * Z);
  if (!e) e = alloc(&p->n_placements, F);
  if (!e) e = alloc(&p->placements, F * Z);
  if (!e) e = alloc(&p->n_canvases, F);
  if (!e) e = alloc(&p->canvas_base, F + 1);
  if (!e) e = alloc(&p->jobs, F * p->job_cap);
  if (!e) e = alloc(&p->canvas_jobs, F * Z);
  if (!e) e = alloc(&p->ranges, static_cast<size_t>(q.max_canvases));
  if (!e) e = alloc(&p->gather_units, 3);
  if (!e) e = alloc(&p->id_state, 1);
  if (!e) e = alloc(&p->look, F);
  if (!e) e = alloc(&p->psync, 3);
  if (!e) e = cudaMemset(p->id_state, 0, sizeof(uint64_t));
  if (!e) e = cudaMemset(p->look, 0, F * sizeof(uint64_t));
  if (!e) e = cudaMemset(p->psync, 0, 3 * sizeof(uint32_t));
  if (!e) e = cudaMemset(p->gather_units, 0, 3 * sizeof(int32_t));
  // the initial memsets run on the legacy stream; the pipeline's work runs
  // on non-blocking streams, which do not wait for it
  if (!e) e = cudaDeviceSynchronize();
  if (e) {
    tg_pipeline_destroy(p);
    return cuda_fail(e, "pipeline allocation");
  }
  *out = p;
  return TG_OK;
}

static const uint32_t* raw_zero(const tg_pipeline* p) {
  return p->raw + static_cast<size_t>(p->p.max_frames) * p->p.height * p->mask_words;
}

// the split launches' word flags (null: dense raw bitmap, kernels.cuh)
static uint32_t* raw_flags(const tg_pipeline* p) {
  if (!raw_flag_words(p->p.width)) return nullptr;
  return p->raw + static_cast<size_t>(p->p.max_frames + 1) * p->p.height * p->mask_words;
}

tg_status tg_pipeline_stage_mask_fg(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                    const uint8_t* const* d_prev, void* stream) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  if (n_frames > 0 && (!d_cur || !d_prev))
    return fail(TG_ERR_INVALID_ARGUMENT, "null frame pointer table");
  TG_CUDA(launch_mask_fg(d_cur, d_prev, n_frames, p->p.width, p->p.height, p->p.pitch,
                         p->p.threshold, p->raw, raw_flags(p), p->ctx->sms,
                         pick(p->ctx, stream)));
  return TG_OK;
}

tg_status tg_pipeline_stage_mask_cells(tg_pipeline* p, int32_t n_frames, void* stream) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  TG_CUDA(launch_dilate_cells(p->raw, raw_zero(p), raw_flags(p), n_frames, p->p.width, p->p.height,
                              p->p.dilate_radius,
                              p->cells, p->active, p->p.keep_mask ? p->mask : nullptr,
                              pick(p->ctx, stream)));
  p->last_frames = n_frames;
  return TG_OK;
}

tg_status tg_pipeline_stage_mask(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                 const uint8_t* const* d_prev, void* stream) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  if (n_frames > 0 && (!d_cur || !d_prev))
    return fail(TG_ERR_INVALID_ARGUMENT, "null frame pointer table");
  // K1 + K1b in one cooperative launch; separate launches if the device
  // cannot co-schedule one K1 CTA per SM (e.g. a shared GPU).
  const cudaError_t e = launch_mask_fused(
      d_cur, d_prev, n_frames, p->p.width, p->p.height, p->p.pitch, p->p.threshold,
      p->p.dilate_radius, p->raw, raw_zero(p), raw_flags(p), p->cells, p->active,
      p->p.keep_mask ? p->mask : nullptr,
      p->mask_sync, p->ctx->sms, pick(p->ctx, stream));
  if (e == cudaSuccess) {
    p->last_frames = n_frames;
    if (n_frames > 0) ++p->stats.mask_fused_launches;
    return TG_OK;
  }
  if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported)
    return cuda_fail(e, "launch_mask_fused");
  cudaGetLastError();
  s = tg_pipeline_stage_mask_fg(p, n_frames, d_cur, d_prev, stream);
  if (!s) s = tg_pipeline_stage_mask_cells(p, n_frames, stream);
  if (!s && n_frames > 0) ++p->stats.mask_split_launches;
  return s;
}

tg_status tg_pipeline_stage_plan(tg_pipeline* p, int32_t n_frames, const uint64_t* d_frame_ids,
                                 const int64_t* d_gen_us, uint64_t first_patch_id, void* stream) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  cudaStream_t st = pick(p->ctx, stream);
  PlanArgs a;
  a.n_frames = n_frames;
  a.W = p->p.width;
  a.H = p->p.height;
  a.X = p->p.partition.zones_x;
  a.Y = p->p.partition.zones_y;
  a.M = p->p.canvas.width;
  a.N = p->p.canvas.height;
  a.cells_x = p->cells_x;
  a.cells_y = p->cells_y;
  a.act_words = p->act_words;
  a.max_rois = p->p.max_rois_per_frame;
  a.job_cap = p->job_cap;
  a.bpp = p->p.bytes_per_pixel;
  a.slo_us = p->p.slo_us;
  a.cells = p->cells;
  a.active = p->active;
  a.frame_ids = d_frame_ids;
  a.gen_us = d_gen_us;
  a.n_rois = p->n_rois;
  a.rois = p->rois;
  a.n_patches = p->n_patches;
  a.patches = p->patches;
  a.admitted = p->admitted;
  a.n_placements = p->n_placements;
  a.placements = p->placements;
  a.n_canvases = p->n_canvases;
  a.jobs = p->jobs;
  a.canvas_jobs = p->canvas_jobs;
  a.err = p->ctx->d_err;
  a.first_id = first_patch_id;
  a.max_canvases = p->p.max_canvases;
  a.nbands = p->nbands;
  a.canvas_base = p->canvas_base;
  a.ranges = p->ranges;
  a.gather_units = p->gather_units;
  a.id_state = p->id_state;
  a.look = p->look;
  a.look_cap = p->p.max_frames;
  a.psync = p->psync;
  a.desc_head = p->desc_head;
  a.desc = p->desc_head ? reinterpret_cast<tg_descriptor*>(p->desc_head + 1) : nullptr;
  a.desc_cap = p->desc_cap;
  a.desc_cameras = p->desc_cameras;
  a.desc_fpc = p->desc_fpc;
  TG_CUDA(launch_plan(a, st));
  p->last_frames = n_frames;
  return TG_OK;
}

tg_status tg_pipeline_stage_gather(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                   uint8_t* d_canvases, void* stream) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  if (p->p.max_canvases > 0 && !d_canvases)
    return fail(TG_ERR_INVALID_ARGUMENT, "null canvas buffer");
  if (p->p.max_canvases == 0) return TG_OK;
  GatherArgs g;
  g.frames = d_cur;
  g.pitch = p->p.pitch;
  g.M = p->p.canvas.width;
  g.N = p->p.canvas.height;
  g.nbands = p->nbands;
  g.band = kGatherDefaultBand;
  g.jobs = p->jobs;
  g.ranges = p->ranges;
  g.units = p->gather_units;
  g.out = d_canvases;
  TG_CUDA(launch_gather(g, p->ctx->sms, 0, pick(p->ctx, stream)));
  return TG_OK;
}

tg_status tg_pipeline_run(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                          const uint8_t* const* d_prev, const uint64_t* d_frame_ids,
                          const int64_t* d_gen_us, uint64_t first_patch_id,
                          uint8_t* d_canvases, void* stream) {
  if (!p) return fail(TG_ERR_INVALID_ARGUMENT, "null pipeline");
  tg_status s = tg_pipeline_stage_mask(p, n_frames, d_cur, d_prev, stream);
  if (!s) s = tg_pipeline_stage_plan(p, n_frames, d_frame_ids, d_gen_us, first_patch_id, stream);
  if (!s) s = tg_pipeline_stage_gather(p, n_frames, d_cur, d_canvases, stream);
  return s;
}

tg_status tg_pipeline_graph_create(tg_pipeline* p, int32_t n_frames, const uint8_t* const* d_cur,
                                   const uint8_t* const* d_prev, const uint64_t* d_frame_ids,
                                   const int64_t* d_gen_us, uint64_t first_patch_id,
                                   uint8_t* d_canvases, void* stream, tg_graph** out) {
  *out = nullptr;
  tg_status s = use_device(p->ctx);
  if (s) return s;
  cudaStream_t st = pick(p->ctx, stream);
  tg_graph* g = new tg_graph();
  TG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  s = tg_pipeline_run(p, n_frames, d_cur, d_prev, d_frame_ids, d_gen_us, first_patch_id,
                      d_canvases, st);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &graph);
  if (s) {
    if (graph) cudaGraphDestroy(graph);
    delete g;
    return s;
  }
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "cudaStreamEndCapture");
  }
  g->graph = graph;
  const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
  if (ie != cudaSuccess) {
    cudaGraphDestroy(graph);
    delete g;
    return cuda_fail(ie, "cudaGraphInstantiate");
  }
  *out = g;
  return TG_OK;
}

tg_status tg_graph_launch(tg_graph* g, void* stream) {
  if (!g) return fail(TG_ERR_INVALID_ARGUMENT, "null graph");
  TG_CUDA(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
  return TG_OK;
}

void tg_graph_destroy(tg_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

tg_status tg_pipeline_device_views(tg_pipeline* p, tg_pipeline_views* v) {
  if (!p) return fail(TG_ERR_INVALID_ARGUMENT, "null pipeline");
  v->n_rois = p->n_rois;
  v->rois = p->rois;
  v->n_patches = p->n_patches;
  v->patches = p->patches;
  v->admitted = p->admitted;
  v->n_placements = p->n_placements;
  v->placements = p->placements;
  v->n_canvases = p->n_canvases;
  v->canvas_base = p->canvas_base;
  v->cells = p->cells;
  v->mask = p->mask;
  v->zones = p->zones;
  v->cells_x = p->cells_x;
  v->cells_y = p->cells_y;
  v->mask_words = p->mask_words;
  return TG_OK;
}

size_t tg_descriptor_block_bytes(int64_t cap) {
  static_assert(sizeof(tg_descriptor) == 80 && sizeof(tg_descriptor_header) == 80,
                "descriptor records and headers are 80 bytes");
  return sizeof(tg_descriptor_header) + static_cast<size_t>(cap < 0 ? 0 : cap) * sizeof(tg_descriptor);
}

tg_status tg_pipeline_set_descriptor_output(tg_pipeline* p, void* d_block, int64_t cap,
                                            const int32_t* d_cameras, int32_t frames_per_camera) {
  if (!p) return fail(TG_ERR_INVALID_ARGUMENT, "null pipeline");
  if (d_block && (cap < 0 || (d_cameras && frames_per_camera < 1)))
    return fail(TG_ERR_INVALID_ARGUMENT, "descriptor output needs cap >= 0 and frames_per_camera >= 1");
  if (reinterpret_cast<uintptr_t>(d_block) % 16)
    return fail(TG_ERR_INVALID_ARGUMENT, "descriptor block must be 16-byte aligned");
  p->desc_head = static_cast<tg_descriptor_header*>(d_block);
  p->desc_cap = d_block ? cap : 0;
  p->desc_cameras = d_block ? d_cameras : nullptr;
  p->desc_fpc = d_block && d_cameras ? frames_per_camera : 1;
  return TG_OK;
}

tg_status tg_pipeline_get_stats(tg_pipeline* p, tg_pipeline_stats* out) {
  if (!p || !out) return fail(TG_ERR_INVALID_ARGUMENT, "null pipeline or output");
  *out = p->stats;
  return TG_OK;
}

tg_status tg_pipeline_download(tg_pipeline* p, int32_t n_frames, void* stream, int32_t* n_rois,
                               tg_rect* rois, int32_t* n_patches, tg_patch_meta* patches,
                               uint8_t* admitted, int32_t* n_placements, tg_placement* placements,
                               int32_t* n_canvases, int64_t* total_canvases) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (n_frames < 0 || n_frames > p->p.max_frames)
    return fail(TG_ERR_INVALID_ARGUMENT, "n_frames must be in [0, max_frames]");
  cudaStream_t st = pick(p->ctx, stream);
  TG_CUDA(cudaStreamSynchronize(st));
  if ((s = check_device_error(p->ctx))) return s;
  const size_t F = n_frames, Z = p->zones;
  if (F == 0) {
    if (total_canvases) *total_canvases = 0;
    return TG_OK;
  }
  if (n_rois) TG_CUDA(cudaMemcpy(n_rois, p->n_rois, 4 * F, cudaMemcpyDeviceToHost));
  if (rois)
    TG_CUDA(cudaMemcpy(rois, p->rois, sizeof(tg_rect) * F * p->p.max_rois_per_frame,
                       cudaMemcpyDeviceToHost));
  if (n_patches) TG_CUDA(cudaMemcpy(n_patches, p->n_patches, 4 * F, cudaMemcpyDeviceToHost));
  if (patches)
    TG_CUDA(cudaMemcpy(patches, p->patches, sizeof(tg_patch_meta) * F * Z, cudaMemcpyDeviceToHost));
  if (admitted) TG_CUDA(cudaMemcpy(admitted, p->admitted, F * Z, cudaMemcpyDeviceToHost));
  if (n_placements)
    TG_CUDA(cudaMemcpy(n_placements, p->n_placements, 4 * F, cudaMemcpyDeviceToHost));
  if (placements)
    TG_CUDA(cudaMemcpy(placements, p->placements, sizeof(tg_placement) * F * Z,
                       cudaMemcpyDeviceToHost));
  if (n_canvases) TG_CUDA(cudaMemcpy(n_canvases, p->n_canvases, 4 * F, cudaMemcpyDeviceToHost));
  if (total_canvases)
    TG_CUDA(cudaMemcpy(total_canvases, p->canvas_base + F, 8, cudaMemcpyDeviceToHost));
  return TG_OK;
}

tg_status tg_pipeline_free_rects(tg_pipeline* p, int32_t frame, tg_free_rect* out, int32_t cap,
                                 int32_t* n_out) {
  tg_status s = use_device(p->ctx);
  if (s) return s;
  if (frame < 0 || frame >= p->last_frames)
    return fail(TG_ERR_OUT_OF_RANGE, "frame index out of range");
  int32_t nc = 0;
  TG_CUDA(cudaMemcpy(&nc, p->n_canvases + frame, 4, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> cj(std::max(1, nc));
  std::vector<Job> jobs(p->job_cap);
  if (nc > 0)
    TG_CUDA(cudaMemcpy(cj.data(), p->canvas_jobs + static_cast<size_t>(frame) * p->zones, 4 * nc,
                       cudaMemcpyDeviceToHost));
  TG_CUDA(cudaMemcpy(jobs.data(), p->jobs + static_cast<size_t>(frame) * p->job_cap,
                     sizeof(Job) * p->job_cap, cudaMemcpyDeviceToHost));
  std::vector<tg_free_rect> fr;
  for (int c = 0; c < nc; ++c) {
    const int start = cj[c] & 0xffff, cnt = cj[c] >> 16;
    for (int i = start; i < start + cnt; ++i) {
      const Job& J = jobs[i];
      if (J.src_frame >= 0) continue;
      fr.push_back(tg_free_rect{tg_rect{J.dx, J.dy, J.w, J.h}, c,
                                static_cast<int32_t>(J.sx | (static_cast<uint32_t>(J.sy) << 16))});
    }
  }
  std::sort(fr.begin(), fr.end(), [](const tg_free_rect& x, const tg_free_rect& y) {
    return x.canvas_index != y.canvas_index ? x.canvas_index < y.canvas_index : x.seq < y.seq;
  });
  *n_out = static_cast<int32_t>(fr.size());
  if (static_cast<int32_t>(fr.size()) > cap) return fail(TG_ERR_CAPACITY, "free rect buffer too small");
  std::copy(fr.begin(), fr.end(), out);
  return TG_OK;
}

// ---- synthetic workload ----------------------------------------------------------
tg_status tg_workload_default(tg_workload_config* c) {
  // trace.hpp:146-160
  c->n_frames = 150;
  c->fps = 15.0;
  c->frame_width = 1920;
  c->frame_height = 1080;
  c->roi_proportion_mean = 0.10;
  c->roi_proportion_jitter = 0.5;
  c->burst_probability = 0.05;
  c->burst_multiplier = 3.0;
  c->roi_count_min = 2;
  c->roi_count_max = 12;
  c->roi_aspect_min = 0.5;
  c->roi_aspect_max = 2.0;
  c->roi_max_dim = 480;
  c->seed = 1;
  return TG_OK;
}

uint64_t tg_derive_seed(uint64_t master, const char* component) {
  // rng.hpp:27-38: FNV-1a of the name, splitmix64 finish.
  uint64_t h = 0xcbf29ce484222325ull;
  for (const unsigned char* q = reinterpret_cast<const unsigned char*>(component); *q; ++q) {
    h ^= *q;
    h *= 0x100000001b3ull;
  }
  uint64_t z = master + 0x9e3779b97f4a7c15ull + h;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

tg_status tg_generate_trace(const tg_workload_config* cfg, int64_t* t_us, int32_t* roi_counts,
                            tg_rect* rois, int64_t roi_cap, int64_t* n_rois_total) {
  const tg_workload_config& c = *cfg;
  // trace.hpp:162-181 validation, same messages.
  if (c.n_frames < 0) return fail(TG_ERR_INVALID_ARGUMENT, "frame count must be >= 0");
  if (!(c.fps > 0.0)) return fail(TG_ERR_INVALID_ARGUMENT, "fps must be positive");
  if (c.frame_width < 1 || c.frame_height < 1)
    return fail(TG_ERR_INVALID_ARGUMENT, "frame dimensions must be positive");
  if (!(c.roi_proportion_mean > 0.0) || c.roi_proportion_mean >= 1.0)
    return fail(TG_ERR_INVALID_ARGUMENT, "roi proportion must be in (0, 1)");
  if (c.roi_proportion_jitter < 0.0 || c.roi_proportion_jitter > 1.0)
    return fail(TG_ERR_INVALID_ARGUMENT, "roi jitter must be in [0, 1]");
  if (c.burst_probability < 0.0 || c.burst_probability > 1.0)
    return fail(TG_ERR_INVALID_ARGUMENT, "burst probability must be in [0, 1]");
  if (c.burst_multiplier < 1.0) return fail(TG_ERR_INVALID_ARGUMENT, "burst multiplier must be >= 1");
  if (c.roi_count_min < 0 || c.roi_count_max < c.roi_count_min)
    return fail(TG_ERR_INVALID_ARGUMENT, "bad roi count range");
  if (!(c.roi_aspect_min > 0.0) || c.roi_aspect_max < c.roi_aspect_min)
    return fail(TG_ERR_INVALID_ARGUMENT, "bad roi aspect range");
  if (c.roi_max_dim < 4) return fail(TG_ERR_INVALID_ARGUMENT, "roi max dim must be >= 4");
  if (c.roi_count_max > 0 && (c.frame_width < 4 || c.frame_height < 4))
    return fail(TG_ERR_INVALID_ARGUMENT, "cannot place requested roi count in frame");
  // rng.hpp:42-70: std::mt19937_64 with hand-rolled distributions.
  std::mt19937_64 eng(tg_derive_seed(c.seed, "trace"));
  auto u01 = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  auto uni = [&](double lo, double hi) { return lo + (hi - lo) * u01(); };
  auto uint_ = [&](int64_t lo, int64_t hi) {
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    return lo + static_cast<int64_t>(eng() % span);
  };
  int64_t total = 0;
  std::vector<double> weights;
  for (int i = 0; i < c.n_frames; ++i) {
    t_us[i] = std::llround(static_cast<double>(i) * 1e6 / c.fps);
    const int W = c.frame_width, H = c.frame_height;
    const bool burst = u01() < c.burst_probability;
    const double jitter = uni(-1.0, 1.0) * c.roi_proportion_jitter;
    double prop = c.roi_proportion_mean * (1.0 + jitter);
    if (burst) prop *= c.burst_multiplier;
    prop = std::clamp(prop, 0.0, 0.6);
    const int n = static_cast<int>(uint_(c.roi_count_min, c.roi_count_max));
    roi_counts[i] = 0;
    if (n > 0 && prop > 0.0) {
      weights.assign(n, 0.0);
      double tw = 0.0;
      for (double& w : weights) {
        w = uni(0.5, 1.5);
        tw += w;
      }
      const double total_area = prop * static_cast<double>(W) * static_cast<double>(H);
      const int max_w = std::min(c.roi_max_dim, W), max_h = std::min(c.roi_max_dim, H);
      for (int r = 0; r < n; ++r) {
        const double area = total_area * weights[r] / tw;
        const double aspect = uni(c.roi_aspect_min, c.roi_aspect_max);
        int w = static_cast<int>(std::lround(std::sqrt(area * aspect)));
        int h = static_cast<int>(std::lround(std::sqrt(area / aspect)));
        w = std::clamp(w, 4, max_w);
        h = std::clamp(h, 4, max_h);
        const int x = static_cast<int>(uint_(0, W - w));
        const int y = static_cast<int>(uint_(0, H - h));
        if (total >= roi_cap) return fail(TG_ERR_CAPACITY, "roi buffer too small");
        rois[total++] = tg_rect{x, y, w, h};
        ++roi_counts[i];
      }
    }
  }
  if (n_rois_total) *n_rois_total = total;
  return TG_OK;
}

tg_status tg_synth_frames(tg_ctx* ctx, int32_t width, int32_t height, int32_t pitch,
                          uint64_t pixel_seed, int32_t n_frames, int32_t t0,
                          const tg_rect* d_rects, const int32_t* d_rect_offsets,
                          uint8_t* const* d_frames, void* stream) {
  tg_status s = use_device(ctx);
  if (s) return s;
  if (width < 16 || width % 16 || pitch < 3 * width || pitch % 16)
    return fail(TG_ERR_INVALID_ARGUMENT, "bad frame geometry");
  SynthArgs a;
  a.W = width;
  a.H = height;
  a.pitch = pitch;
  a.t0 = t0;
  a.seed = pixel_seed;
  a.rects = d_rects;
  a.offsets = d_rect_offsets;
  a.frames = d_frames;
  TG_CUDA(launch_synth(a, n_frames, pick(ctx, stream)));
  return TG_OK;
}

}  // extern "C"
