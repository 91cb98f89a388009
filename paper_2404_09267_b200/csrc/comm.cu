// comm.cu -- the path's only collective: the all-gather of per-rank patch
// descriptor blocks.
//
// Cameras are sharded over GPUs in contiguous blocks, so the rank-major
// concatenation of the ranks' blocks is the reference's camera-major patch
// list (sim.hpp:241-262); the batcher consumes it on the host.  Pixels never
// cross GPUs here.  Two transports behind one handle:
//   - device: NCCL (ncclAllGather over NVLink / NVSwitch, opened at run
//     time) on device
//     buffers, stream-ordered -- one call gathers every rank's block with
//     its record count in the header, so no separate count exchange and no
//     host sync;
//   - host: a caller-supplied all-gather over host buffers (tests drive the
//     multi-rank logic through it on CPU; any out-of-band transport works).
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "kernels.cuh"
#include "tangram_gpu.h"

extern "C" void tg_internal_set_error(const char* msg);
extern "C" int tg_internal_ctx_device(tg_ctx* ctx);

struct tg_comm {
  int rank = 0, world = 1, device = -1;
  ncclComm_t nccl = nullptr;
  tg_host_allgather_fn fn = nullptr;
  void* user = nullptr;
};

namespace {

// NCCL is opened on first use, not linked: loading the library must not pull
// a libnccl.so.2 into the process before a framework that ships its own
// (newer) one (PyTorch binds to whichever copy of the soname is loaded
// first).  Preference: a libnccl.so.2 already in the process, then
// $TG_NCCL_LIB, then the system's.
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = std::getenv("TG_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      const char* e = dlerror();
      api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [h](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy ||
        !api.error_string) {
      api.error = "libnccl.so.2 lacks a required symbol";
      return;
    }
    api.handle = h;
  });
  return api;
}

tg_status comm_fail(tg_status s, const char* what, const char* why) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: %s", what, why);
  tg_internal_set_error(buf);
  return s;
}

tg_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return TG_OK;
  return comm_fail(TG_ERR_COMM, what, nccl().error_string(r));
}

tg_status nccl_loaded(const char* what) {
  return nccl().handle ? TG_OK : comm_fail(TG_ERR_COMM, what, nccl().error.c_str());
}

}  // namespace

extern "C" {

tg_status tg_comm_get_unique_id(tg_comm_id* out) {
  static_assert(sizeof(ncclUniqueId) == sizeof(tg_comm_id), "tg_comm_id mirrors ncclUniqueId");
  tg_status s = nccl_loaded("tg_comm_get_unique_id");
  if (s) return s;
  ncclUniqueId id;
  s = nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  if (s) return s;
  memcpy(out->bytes, &id, sizeof(id));
  return TG_OK;
}

tg_status tg_comm_create(tg_ctx* ctx, const tg_comm_id* id, int32_t rank, int32_t world,
                         tg_comm** out) {
  *out = nullptr;
  if (!ctx || !id) return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_create", "null argument");
  if (world < 1 || rank < 0 || rank >= world)
    return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_create", "need 0 <= rank < world");
  if (tg_status ls = nccl_loaded("tg_comm_create")) return ls;
  const int dev = tg_internal_ctx_device(ctx);
  if (cudaSetDevice(dev) != cudaSuccess)
    return comm_fail(TG_ERR_NO_DEVICE, "tg_comm_create", "no CUDA device");
  ncclUniqueId uid;
  memcpy(&uid, id->bytes, sizeof(uid));
  tg_comm* c = new tg_comm();
  c->rank = rank;
  c->world = world;
  c->device = dev;
  const tg_status s =
      nccl_check(nccl().comm_init_rank(&c->nccl, world, uid, rank), "ncclCommInitRank");
  if (s) {
    delete c;
    return s;
  }
  *out = c;
  return TG_OK;
}

tg_status tg_comm_create_host(int32_t rank, int32_t world, tg_host_allgather_fn fn, void* user,
                              tg_comm** out) {
  *out = nullptr;
  if (!fn) return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_create_host", "null all-gather");
  if (world < 1 || rank < 0 || rank >= world)
    return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_create_host", "need 0 <= rank < world");
  tg_comm* c = new tg_comm();
  c->rank = rank;
  c->world = world;
  c->fn = fn;
  c->user = user;
  *out = c;
  return TG_OK;
}

void tg_comm_destroy(tg_comm* comm) {
  if (!comm) return;
  if (comm->nccl) {
    cudaSetDevice(comm->device);
    nccl().comm_destroy(comm->nccl);
  }
  delete comm;
}

tg_status tg_comm_info(tg_comm* comm, int32_t* rank, int32_t* world, int32_t* on_device) {
  if (!comm) return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_info", "null communicator");
  if (rank) *rank = comm->rank;
  if (world) *world = comm->world;
  if (on_device) *on_device = comm->nccl ? 1 : 0;
  return TG_OK;
}

tg_status tg_comm_allgather(tg_comm* comm, const void* send, size_t bytes, void* recv,
                            void* stream) {
  if (!comm) return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_allgather", "null communicator");
  if (bytes > 0 && (!send || !recv))
    return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_comm_allgather", "null buffer");
  if (comm->nccl) {
    if (cudaSetDevice(comm->device) != cudaSuccess)
      return comm_fail(TG_ERR_CUDA, "tg_comm_allgather", "cudaSetDevice");
    return nccl_check(nccl().all_gather(send, recv, bytes, ncclUint8, comm->nccl,
                                        static_cast<cudaStream_t>(stream)),
                      "ncclAllGather");
  }
  if (comm->fn(send, bytes, recv, comm->user) != 0)
    return comm_fail(TG_ERR_COMM, "tg_comm_allgather", "host transport failed");
  return TG_OK;
}

tg_status tg_descriptors_allgather(tg_comm* comm, const void* block, int64_t cap,
                                   void* blocks_out, void* stream) {
  if (cap < 0) return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_descriptors_allgather", "cap < 0");
  return tg_comm_allgather(comm, block, tg_descriptor_block_bytes(cap), blocks_out, stream);
}

tg_status tg_descriptor_blocks_flatten(const void* blocks, int32_t n_blocks, int64_t cap,
                                       tg_descriptor* out, int64_t out_cap, int64_t* n_out) {
  *n_out = 0;
  if (n_blocks < 0 || cap < 0)
    return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_descriptor_blocks_flatten", "bad block layout");
  const size_t bb = tg_descriptor_block_bytes(cap);
  int64_t k = 0;
  for (int32_t r = 0; r < n_blocks; ++r) {
    const char* b = static_cast<const char*>(blocks) + static_cast<size_t>(r) * bb;
    tg_descriptor_header h;
    memcpy(&h, b, sizeof(h));
    if (h.count < 0 || h.count > cap) {
      char why[128];
      snprintf(why, sizeof(why), "block %d holds %lld records (cap %lld)", r,
               static_cast<long long>(h.count), static_cast<long long>(cap));
      return comm_fail(TG_ERR_INVALID_ARGUMENT, "tg_descriptor_blocks_flatten", why);
    }
    if (k + h.count > out_cap)
      return comm_fail(TG_ERR_CAPACITY, "tg_descriptor_blocks_flatten", "output too small");
    memcpy(out + k, b + sizeof(tg_descriptor_header), static_cast<size_t>(h.count) * sizeof(tg_descriptor));
    k += h.count;
  }
  *n_out = k;
  return TG_OK;
}

}  // extern "C"
