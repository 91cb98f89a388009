// Green-context feasibility probe: split the device's SMs into two partitions,
// launch runtime (<<<>>>) kernels on a stream of each, check where the CTAs
// ran (%smid) and the read bandwidth a partition reaches alone and beside
// the other.  Tuning aid, not part of the product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("%s: %s\n", #x, s); exit(1);} } while (0)
#define CR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(r_)); exit(1);} } while (0)

__global__ void smids(int* out) {
  if (threadIdx.x == 0) { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); out[blockIdx.x] = s; }
}
__global__ void readk(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  int want = argc > 1 ? atoi(argv[1]) : 16;
  CR(cudaSetDevice(0));
  CR(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  CUdevResource small_[1], rest; unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(small_, &ng, &all, &rest, 0, want));
  printf("split: small %u SMs (groups %u), rest %u SMs\n", small_[0].sm.smCount, ng, rest.sm.smCount);
  CUdevResourceDesc dA, dB; CK(cuDevResourceGenerateDesc(&dA, &rest, 1)); CK(cuDevResourceGenerateDesc(&dB, &small_[0], 1));
  CUgreenCtx gA, gB; CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB; CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  int* d; CR(cudaMalloc(&d, 4096 * sizeof(int)));
  std::vector<int> h(4096);
  for (int which = 0; which < 2; ++which) {
    cudaStream_t s = (cudaStream_t)(which ? sB : sA);
    CR(cudaMemset(d, 0xff, 4096 * 4));
    smids<<<1024, 32, 0, s>>>(d);
    CR(cudaGetLastError()); CR(cudaStreamSynchronize(s));
    CR(cudaMemcpy(h.data(), d, 4096 * 4, cudaMemcpyDeviceToHost));
    std::vector<int> seen(256, 0); int n = 0;
    for (int i = 0; i < 1024; ++i) if (h[i] >= 0 && !seen[h[i]]++) ++n;
    printf("partition %c: CTAs ran on %d distinct SMs\n", which ? 'B' : 'A', n);
  }
  size_t bytes = size_t(8) << 30; uint4* buf; CR(cudaMalloc(&buf, bytes)); CR(cudaMemset(buf, 1, bytes));
  unsigned* sink; CR(cudaMalloc(&sink, 4));
  size_t n = bytes / 16;
  cudaEvent_t e0, e1; CR(cudaEventCreate(&e0)); CR(cudaEventCreate(&e1));
  auto run = [&](cudaStream_t s, int grid, const char* name) {
    readk<<<grid, 1024, 0, s>>>(buf, n, sink);
    CR(cudaEventRecord(e0, s));
    for (int i = 0; i < 3; ++i) readk<<<grid, 1024, 0, s>>>(buf, n, sink);
    CR(cudaEventRecord(e1, s)); CR(cudaEventSynchronize(e1));
    float ms; CR(cudaEventElapsedTime(&ms, e0, e1));
    printf("%s: %.1f GB/s\n", name, 3.0 * bytes / (ms / 1e3) / 1e9);
  };
  run((cudaStream_t)0, all.sm.smCount * 2, "whole device (default stream)");
  run((cudaStream_t)sA, rest.sm.smCount * 2, "partition A alone");
  run((cudaStream_t)sB, small_[0].sm.smCount * 2, "partition B alone");
  return 0;
}
