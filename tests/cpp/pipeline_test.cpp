// pipeline_test.cpp -- the hot path driven from C++ through the C ABI alone
// (no Python): synthetic camera frames on the device -> tg_pipeline_run ->
// device descriptor block -> NCCL all-gather (world size 1) -> SLO batcher
// (tg_batcher_schedule) -> event canvases (tg_batcher_gather_all).  Every per-frame result and canvas byte is checked
// against the plain-C oracle (oracle/tangram_oracle.c, test infrastructure)
// on the same frames; the batcher's canvases against a host fill of its own
// placements.  Built by tests/cpp/Makefile; run by tests/test_gpu_parity.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../oracle/tangram_oracle.h"
#include "tangram_gpu.h"

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)
#define OK(call)                                                                  \
  do {                                                                            \
    const tg_status s_ = (call);                                                  \
    if (s_ != TG_OK) {                                                            \
      std::printf("FAIL %s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, s_,   \
                  tg_last_error());                                               \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

int main() {
  const int W = 1920, H = 1080, n = 10, pitch = 3 * W, C = 3;
  const size_t fb = static_cast<size_t>(pitch) * H;
  tg_ctx* ctx = nullptr;
  OK(tg_ctx_create(0, &ctx));

  // ---- synthetic camera: generator RoIs (trace.hpp:184-231) -> device frames
  tg_workload_config wc;
  OK(tg_workload_default(&wc));
  wc.n_frames = n;
  wc.fps = 30.0;
  wc.frame_width = W;
  wc.frame_height = H;
  wc.roi_proportion_mean = 0.15;
  wc.seed = 1000;
  std::vector<int64_t> t_us(n);
  std::vector<int32_t> counts(n);
  std::vector<tg_rect> rects(static_cast<size_t>(n) * wc.roi_count_max);
  int64_t n_rects = 0;
  OK(tg_generate_trace(&wc, t_us.data(), counts.data(), rects.data(),
                       static_cast<int64_t>(rects.size()), &n_rects));
  std::vector<int32_t> offs(n + 2, 0);  // [0, 0] background, then frame i at offs[i+1]
  for (int i = 0; i < n; ++i) offs[i + 2] = offs[i + 1] + counts[i];
  uint8_t* ring = nullptr;
  OK(tg_malloc_device(ctx, fb * (n + 1), reinterpret_cast<void**>(&ring)));
  std::vector<uint8_t*> slots(n + 1);
  for (int i = 0; i <= n; ++i) slots[i] = ring + fb * i;
  tg_rect* d_rects = nullptr;
  int32_t* d_offs = nullptr;
  uint8_t** d_slots = nullptr;
  OK(tg_malloc_device(ctx, sizeof(tg_rect) * (n_rects + 1), reinterpret_cast<void**>(&d_rects)));
  OK(tg_malloc_device(ctx, sizeof(int32_t) * offs.size(), reinterpret_cast<void**>(&d_offs)));
  OK(tg_malloc_device(ctx, sizeof(uint8_t*) * slots.size(), reinterpret_cast<void**>(&d_slots)));
  OK(tg_memcpy_async(ctx, d_rects, rects.data(), sizeof(tg_rect) * n_rects, 0, nullptr));
  OK(tg_memcpy_async(ctx, d_offs, offs.data(), sizeof(int32_t) * offs.size(), 0, nullptr));
  OK(tg_memcpy_async(ctx, d_slots, slots.data(), sizeof(uint8_t*) * slots.size(), 0, nullptr));
  const uint64_t pixel_seed = tg_derive_seed(1000, "pixels");
  OK(tg_synth_frames(ctx, W, H, pitch, pixel_seed, 1, -1, d_rects, d_offs, d_slots, nullptr));
  OK(tg_synth_frames(ctx, W, H, pitch, pixel_seed, n, 0, d_rects, d_offs + 1, d_slots + 1, nullptr));

  // ---- the per-frame path ------------------------------------------------
  tg_pipeline_params pp;
  OK(tg_pipeline_params_default(W, H, &pp));
  pp.max_frames = n;
  pp.max_canvases = n * 16;
  tg_pipeline* pipe = nullptr;
  OK(tg_pipeline_create(ctx, &pp, &pipe));
  std::vector<uint64_t> ids(n);
  for (int i = 0; i < n; ++i) ids[i] = static_cast<uint64_t>(i);
  uint64_t* d_ids = nullptr;
  int64_t* d_gen = nullptr;
  uint8_t *d_canv = nullptr, *d_bcanv = nullptr;
  const size_t cb = static_cast<size_t>(pp.canvas.width) * pp.canvas.height * C;
  OK(tg_malloc_device(ctx, 8 * n, reinterpret_cast<void**>(&d_ids)));
  OK(tg_malloc_device(ctx, 8 * n, reinterpret_cast<void**>(&d_gen)));
  OK(tg_malloc_device(ctx, cb * pp.max_canvases, reinterpret_cast<void**>(&d_canv)));
  OK(tg_memcpy_async(ctx, d_ids, ids.data(), 8 * n, 0, nullptr));
  OK(tg_memcpy_async(ctx, d_gen, t_us.data(), 8 * n, 0, nullptr));
  // the planner's dense device descriptor list
  const int64_t dcap = static_cast<int64_t>(n) * pp.partition.zones_x * pp.partition.zones_y;
  const size_t bb = tg_descriptor_block_bytes(dcap);
  void *d_block = nullptr, *d_blocks = nullptr;
  int32_t* d_cams = nullptr;
  const int32_t cam_ids[1] = {7};
  OK(tg_malloc_device(ctx, bb, &d_block));
  OK(tg_malloc_device(ctx, bb, &d_blocks));
  OK(tg_malloc_device(ctx, sizeof(cam_ids), reinterpret_cast<void**>(&d_cams)));
  OK(tg_memcpy_async(ctx, d_cams, cam_ids, sizeof(cam_ids), 0, nullptr));
  OK(tg_pipeline_set_descriptor_output(pipe, d_block, dcap, d_cams, n));
  OK(tg_pipeline_run(pipe, n, d_slots + 1, d_slots, d_ids, d_gen, 0, d_canv, nullptr));
  // the collective: NCCL all-gather of the descriptor blocks (one rank here)
  tg_comm_id cid;
  OK(tg_comm_get_unique_id(&cid));
  tg_comm* comm = nullptr;
  OK(tg_comm_create(ctx, &cid, 0, 1, &comm));
  int32_t c_rank = -1, c_world = 0, c_dev = 0;
  OK(tg_comm_info(comm, &c_rank, &c_world, &c_dev));
  CHECK(c_rank == 0 && c_world == 1 && c_dev == 1);
  OK(tg_descriptors_allgather(comm, d_block, dcap, d_blocks, tg_ctx_stream(ctx)));
  std::vector<uint8_t> hblocks(bb);
  OK(tg_memcpy_async(ctx, hblocks.data(), d_blocks, bb, 1, nullptr));

  tg_pipeline_views v;
  OK(tg_pipeline_device_views(pipe, &v));
  const int Z = v.zones;
  std::vector<int32_t> n_rois(n), n_patches(n), n_pl(n), n_canv(n);
  std::vector<tg_rect> rois(static_cast<size_t>(n) * pp.max_rois_per_frame);
  std::vector<tg_patch_meta> patches(static_cast<size_t>(n) * Z);
  std::vector<uint8_t> admitted(static_cast<size_t>(n) * Z);
  std::vector<tg_placement> pl(static_cast<size_t>(n) * Z);
  int64_t total = 0;
  OK(tg_pipeline_download(pipe, n, nullptr, n_rois.data(), rois.data(), n_patches.data(),
                          patches.data(), admitted.data(), n_pl.data(), pl.data(), n_canv.data(),
                          &total));
  std::vector<uint8_t> canv(cb * total);
  OK(tg_memcpy_async(ctx, canv.data(), d_canv, canv.size(), 1, nullptr));
  std::vector<uint8_t> host(fb * (n + 1));
  OK(tg_memcpy_async(ctx, host.data(), ring, host.size(), 1, nullptr));
  OK(tg_ctx_synchronize(ctx));

  // ---- the oracle on the same frames ---------------------------------------
  orc_path_params op{W, H, pitch, pp.threshold, pp.dilate_radius, pp.partition.zones_x,
                     pp.partition.zones_y, pp.canvas.width, pp.canvas.height,
                     pp.bytes_per_pixel, pp.slo_us, pp.max_rois_per_frame, 4};
  std::vector<const uint8_t*> cur(n), prev(n);
  for (int i = 0; i < n; ++i) {
    cur[i] = host.data() + fb * (i + 1);
    prev[i] = host.data() + fb * i;
  }
  std::vector<int32_t> o_nr(n), o_np(n), o_nc(n), o_npl(n);
  std::vector<orc_rect> o_rois(rois.size());
  std::vector<orc_patch> o_patches(patches.size());
  std::vector<uint8_t> o_adm(admitted.size());
  std::vector<orc_placement> o_pl(pl.size());
  std::vector<uint8_t> o_canv(cb * pp.max_canvases);
  orc_path_out oo{o_nr.data(), o_rois.data(), o_np.data(), o_patches.data(), o_adm.data(),
                  o_nc.data(), o_pl.data(), o_npl.data(), o_canv.data(), pp.max_canvases,
                  nullptr, 0};
  CHECK(orc_process_frames(&op, n, cur.data(), prev.data(), ids.data(), t_us.data(), 0, &oo) == 0);
  CHECK(total == oo.total_canvases && total > 0);
  for (int i = 0; i < n; ++i) {
    CHECK(n_rois[i] == o_nr[i]);
    for (int r = 0; r < n_rois[i] && r < o_nr[i]; ++r) {
      const tg_rect& a = rois[static_cast<size_t>(i) * pp.max_rois_per_frame + r];
      const orc_rect& b = o_rois[static_cast<size_t>(i) * pp.max_rois_per_frame + r];
      CHECK(a.x == b.x && a.y == b.y && a.w == b.w && a.h == b.h);
    }
    CHECK(n_patches[i] == o_np[i] && n_pl[i] == o_npl[i] && n_canv[i] == o_nc[i]);
    for (int j = 0; j < n_patches[i]; ++j) {
      const tg_patch_meta& a = patches[static_cast<size_t>(i) * Z + j];
      const orc_patch& b = o_patches[static_cast<size_t>(i) * Z + j];
      CHECK(a.patch_id == b.patch_id && a.rect.x == b.rect.x && a.rect.y == b.rect.y &&
            a.rect.w == b.rect.w && a.rect.h == b.rect.h && a.size_bytes == b.size_bytes &&
            a.deadline_us == b.deadline_us);
      CHECK(admitted[static_cast<size_t>(i) * Z + j] == o_adm[static_cast<size_t>(i) * Z + j]);
    }
    for (int k = 0; k < n_pl[i]; ++k) {
      const tg_placement& a = pl[static_cast<size_t>(i) * Z + k];
      const orc_placement& b = o_pl[static_cast<size_t>(i) * Z + k];
      CHECK(a.patch_id == b.patch_id && a.canvas_index == b.canvas_index &&
            a.position.x == b.position.x && a.position.y == b.position.y);
    }
  }
  CHECK(std::memcmp(canv.data(), o_canv.data(), canv.size()) == 0);

  // ---- SLO batcher over the gathered descriptors, canvases on the device ---
  // the device list equals the host compaction of the per-frame slots
  std::vector<tg_descriptor> desc(static_cast<size_t>(n) * Z), hdesc(desc.size());
  int64_t nd = 0, nh = 0;
  const int32_t* cams = cam_ids;
  OK(tg_descriptor_blocks_flatten(hblocks.data(), 1, dcap, desc.data(),
                                  static_cast<int64_t>(desc.size()), &nd));
  OK(tg_descriptors_compact(patches.data(), n_patches.data(), admitted.data(), Z, cams, 1, n,
                            hdesc.data(), static_cast<int64_t>(hdesc.size()), &nh));
  CHECK(nd == nh && nd > 0);
  CHECK(std::memcmp(desc.data(), hdesc.data(), sizeof(tg_descriptor) * nd) == 0);
  const tg_profile_entry prof[4] = {{1, 60.0, 3.0}, {2, 85.0, 4.0}, {4, 135.0, 6.0},
                                    {8, 235.0, 10.0}};
  tg_batcher* b = nullptr;
  OK(tg_batcher_create(pp.canvas, prof, 4, 8, &b));
  std::vector<tg_patch_meta> adm(nd);
  std::vector<int32_t> src(nd);
  std::vector<int64_t> arr(nd);
  int64_t n_adm = 0;
  int32_t n_ev = 0;
  OK(tg_batcher_schedule(b, desc.data(), nd, cams, 1, n, 40.0, 1, adm.data(), src.data(),
                         arr.data(), &n_adm, &n_ev));
  CHECK(n_ev > 0 && n_adm > 0);
  int64_t nbc = 0;
  OK(tg_malloc_device(ctx, cb * n_adm, reinterpret_cast<void**>(&d_bcanv)));
  OK(tg_batcher_gather_all(ctx, b, d_slots, pitch, d_bcanv, n_adm, &nbc, nullptr));
  std::vector<uint8_t> bcanv(cb * nbc);
  OK(tg_memcpy_async(ctx, bcanv.data(), d_bcanv, bcanv.size(), 1, nullptr));
  OK(tg_ctx_synchronize(ctx));
  // host fill of every event's placements (uncovered bytes are zero)
  int64_t k = 0;
  for (int e = 0; e < n_ev; ++e) {
    tg_invoke_info info;
    OK(tg_batcher_event(b, e, &info, nullptr, nullptr, nullptr));
    std::vector<uint64_t> pid(info.n_patches);
    std::vector<tg_placement> epl(info.n_patches);
    OK(tg_batcher_event(b, e, &info, pid.data(), epl.data(), nullptr));
    std::vector<uint8_t> want(cb * info.batch_size, 0);
    for (const tg_placement& p : epl) {
      int64_t q = 0;
      while (q < n_adm && adm[q].patch_id != p.patch_id) ++q;
      CHECK(q < n_adm);
      if (q == n_adm) continue;
      const uint8_t* frame = host.data() + fb * src[q];
      for (int y = 0; y < p.position.h; ++y)
        std::memcpy(want.data() + cb * p.canvas_index +
                        (static_cast<size_t>(p.position.y + y) * pp.canvas.width + p.position.x) * C,
                    frame + static_cast<size_t>(adm[q].rect.y + y) * pitch + adm[q].rect.x * C,
                    static_cast<size_t>(p.position.w) * C);
    }
    CHECK(std::memcmp(bcanv.data() + cb * k, want.data(), want.size()) == 0);
    k += info.batch_size;
  }
  CHECK(k == nbc);

  tg_batcher_destroy(b);
  tg_comm_destroy(comm);
  tg_pipeline_destroy(pipe);
  for (void* ptr : {static_cast<void*>(ring), static_cast<void*>(d_rects),
                    static_cast<void*>(d_offs), static_cast<void*>(d_slots),
                    static_cast<void*>(d_ids), static_cast<void*>(d_gen),
                    static_cast<void*>(d_canv), static_cast<void*>(d_bcanv), d_block, d_blocks,
                    static_cast<void*>(d_cams)})
    OK(tg_free_device(ctx, ptr));
  tg_ctx_destroy(ctx);
  std::printf("%lld per-frame canvases, %d invoke events, %lld event canvases: %s\n",
              static_cast<long long>(total), n_ev, static_cast<long long>(nbc),
              g_fail ? "FAILURES" : "ALL PASS");
  return g_fail ? 1 : 0;
}
