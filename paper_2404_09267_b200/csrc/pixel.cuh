// pixel.cuh -- per-pixel helpers shared by the mask kernels (k_mask.cu,
// k_band.cu): SWAR frame differencing + threshold, cell summary packing,
// mbarrier arrive / test_wait, acquire loads.  Frozen spec: DESIGN.md §3.
#pragma once

#include "common.cuh"

namespace tg {

// Cell summary (frozen spec): bits 0-8 count, 9-12 x0, 13-16 x1, 17-20 y0,
// 21-24 y1 of the dilated foreground inside the 16x16 cell.
__device__ __forceinline__ uint32_t pack_cell(int occ, uint32_t cols, uint32_t rows) {
  if (occ == 0) return 0u;
  const uint32_t x0 = __ffs(cols) - 1, x1 = 31 - __clz(cols);
  const uint32_t y0 = __ffs(rows) - 1, y1 = 31 - __clz(rows);
  return static_cast<uint32_t>(occ) | x0 << 9 | x1 << 13 | y0 << 17 | y1 << 21;
}

// Per-byte "d > T" flag in bit 7 of each byte, SWAR without cross-byte
// borrows.  kLow (T <= 127): t1 = (T+1)*0x01010101; otherwise t1 =
// (T-127)*0x01010101 and only bytes with their top bit set can pass.
template <bool kLow>
__device__ __forceinline__ uint32_t gt_bytes(uint32_t d, uint32_t t1) {
  if (kLow) return d | ((d | 0x80808080u) - t1);
  return d & (((d & 0x7f7f7f7fu) | 0x80808080u) - t1);
}

// 4 pixels (12 bytes) of cur/prev -> 4 foreground bits (max_c |cur-prev| > T
// <=> some channel's |cur-prev| > T).
template <bool kLow>
__device__ __forceinline__ uint32_t fg4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t b0,
                                        uint32_t b1, uint32_t b2, uint32_t t1) {
  const uint32_t g0 = gt_bytes<kLow>(__vabsdiffu4(a0, b0), t1);
  const uint32_t g1 = gt_bytes<kLow>(__vabsdiffu4(a1, b1), t1);
  const uint32_t g2 = gt_bytes<kLow>(__vabsdiffu4(a2, b2), t1);
  // Planar regroup: R=[p0.c0 p1.c0 p2.c0 p3.c0], G=[..c1], B=[..c2].
  const uint32_t r = __byte_perm(__byte_perm(g0, g1, 0x0630), g2, 0x5210);
  const uint32_t g = __byte_perm(__byte_perm(g0, g1, 0x0741), g2, 0x6210);
  const uint32_t b = __byte_perm(__byte_perm(g0, g1, 0x0052), g2, 0x7410);
  // bits 7/15/23/31 -> bits 28..31 with one multiply (no colliding terms).
  return (((r | g | b) & 0x80808080u) * 0x00204081u) >> 28;
}

// 32 pixels (96 bytes as 6 x 16) of cur/prev -> 32 raw foreground bits.
template <bool kLow>
__device__ __forceinline__ uint32_t fg_word(const uint4 (&c)[6], const uint4 (&p)[6], uint32_t t1) {
  uint32_t bits = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint4 c0 = c[3 * h], c1 = c[3 * h + 1], c2 = c[3 * h + 2];
    const uint4 p0 = p[3 * h], p1 = p[3 * h + 1], p2 = p[3 * h + 2];
    uint32_t v = fg4<kLow>(c0.x, c0.y, c0.z, p0.x, p0.y, p0.z, t1);
    v |= fg4<kLow>(c0.w, c1.x, c1.y, p0.w, p1.x, p1.y, t1) << 4;
    v |= fg4<kLow>(c1.z, c1.w, c2.x, p1.z, p1.w, p2.x, t1) << 8;
    v |= fg4<kLow>(c2.y, c2.z, c2.w, p2.y, p2.z, p2.w, t1) << 12;
    bits |= v << (16 * h);
  }
  return bits;
}

__device__ __forceinline__ void load96(uint4 (&v)[6], const uint8_t* p) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = lds128(p + 16 * k);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace tg
