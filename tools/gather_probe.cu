// Microbenchmark: device bandwidth of reading S-byte spans at scattered
// 16-byte-aligned offsets of a large buffer, via (a) per-warp LDG.128 and
// (b) per-warp cp.async.bulk into a shared-memory ring; read-only (values
// folded into a checksum) and read+write (spans copied to a dense output).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void ldg_kernel(const uint8_t* src, const uint64_t* offs, int nspans, int S, uint8_t* dst, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x / 32);
  unsigned acc = 0;
  for (int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < nspans; i += warps) {
    const uint4* s = reinterpret_cast<const uint4*>(src + offs[i]);
    uint4* d = reinterpret_cast<uint4*>(dst + static_cast<size_t>(i) * S);
    for (int c = lane; c < S / 16; c += 32) {
      const uint4 v = __ldg(s + c);
      if (dst) d[c] = v; else acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

constexpr int kSlots = 8;
__global__ void tma_kernel(const uint8_t* src, const uint64_t* offs, int nspans, int S, int slot_bytes, uint8_t* dst, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x / 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm) + warp * kSlots;
  uint8_t* ring = sm + 8 * kSlots * nw + static_cast<size_t>(warp) * kSlots * slot_bytes;
  if (lane < kSlots) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + lane)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int warps = gridDim.x * nw;
  const int first = blockIdx.x * nw + warp;
  int n = first < nspans ? (nspans - first + warps - 1) / warps : 0;
  unsigned acc = 0;
  auto issue = [&](int k) {
    const int slot = k % kSlots;
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + slot)), "r"(S) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + slot * slot_bytes)),
                   "l"(src + offs[first + k * warps]), "r"(S), "r"(smem_u32(bars + slot)) : "memory");
    }
  };
  for (int k = 0; k < kSlots - 1 && k < n; ++k) issue(k);
  for (int k = 0; k < n; ++k) {
    if (k + kSlots - 1 < n) issue(k + kSlots - 1);
    const int slot = k % kSlots;
    const uint32_t par = (k / kSlots) & 1;
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(smem_u32(bars + slot)), "r"(par) : "memory");
    const uint4* s = reinterpret_cast<const uint4*>(ring + slot * slot_bytes);
    uint4* d = dst ? reinterpret_cast<uint4*>(dst + static_cast<size_t>(first + k * warps) * S) : nullptr;
    for (int c = lane; c < S / 16; c += 32) {
      const uint4 v = s[c];
      if (d) d[c] = v; else acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const size_t SRC = 8ull << 30, DST = 2ull << 30;
  uint8_t *src, *dst;
  unsigned* sink;
  CK(cudaMalloc(&src, SRC));
  CK(cudaMalloc(&dst, DST));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(src, 1, SRC));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int spans_S[] = {256, 512, 1024, 2048, 4096, 16384, 65536};
  for (int S : spans_S) {
    const int nspans = static_cast<int>((1ull << 30) / S) ;  // 1 GB read
    std::vector<uint64_t> h(nspans);
    uint64_t x = 88172645463325252ull;
    for (auto& o : h) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      o = (x % ((SRC - S) / 16)) * 16;
    }
    uint64_t* offs;
    CK(cudaMalloc(&offs, nspans * 8));
    CK(cudaMemcpy(offs, h.data(), nspans * 8, cudaMemcpyHostToDevice));
    for (int write = 0; write < 2; ++write) {
      uint8_t* d = write ? dst : nullptr;
      for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9;
        for (int blocks_per_sm : {4, 8}) {
          const int threads = 256;
          const int slot_bytes = S;
          const size_t smem = 8 * kSlots * 8 + static_cast<size_t>(8) * kSlots * slot_bytes;
          if (mode == 1) {
            if (smem > 227 * 1024) continue;
            CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
          }
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0)
              ldg_kernel<<<sms * blocks_per_sm, threads>>>(src, offs, nspans, S, d, sink);
            else
              tma_kernel<<<sms * blocks_per_sm, threads, smem>>>(src, offs, nspans, S, slot_bytes, d, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
          }
        }
        const double bytes = static_cast<double>(nspans) * S * (write ? 2 : 1);
        printf("S=%5d %-4s %-10s %.3f ms  %.0f GB/s\n", S, mode ? "tma" : "ldg", write ? "read+write" : "read", best, bytes / best / 1e6);
      }
    }
    cudaFree(offs);
  }
  return 0;
}
