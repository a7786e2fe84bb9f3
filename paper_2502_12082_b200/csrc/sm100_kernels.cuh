// sm100_kernels.cuh — shared pieces of the tcgen05 / TMEM / TMA kernels of the bf16 hot path (sm_100a).
//
// Every kernel is warp-specialised, one CTA per 128-row block of one head (B_r = B_c = 128): math
// warps with thread ↔ TMEM lane ↔ row (a query row in the τ / output / dQ kernels, a key row in the
// dK/dV kernel), one TMA producer warp (stage ring, mbarrier full/empty) and one MMA-issuer warp that
// owns the TMEM allocation (see sm100_tau.cuh and sm100_fb.cuh for the per-kernel layouts).  Operand
// tiles are [128 rows × 64 bf16] boxes with the 128-byte swizzle, used K-major (contraction over d) or
// MN-major (contraction over rows) by descriptor choice; the operands the math warps produce (P, U,
// dS) go back into TMEM and feed TS-MMAs.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace entmax {
namespace sm100 {

constexpr uint32_t kChunkBytes = 128 * 128;   // one [128 rows × 64 bf16] SW128 box = 16 KB

template <int D>
struct Cfg {
  static constexpr int KCH = D / 64;                        // 64-wide d chunks per tile
  static constexpr uint32_t TILE = 128u * D * 2u;           // bytes of a [128 × D] bf16 tile
  static constexpr int KSTEPS = D / 16;                     // MMA K-steps over d
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return (uint8_t*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

// load one [128 × D] tile (KCH boxes) of head (b,h), rows starting at row0
template <int D>
__device__ __forceinline__ void tma_tile(uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int row0, int h, int b) {
#pragma unroll
  for (int c = 0; c < Cfg<D>::KCH; ++c) ptx::tma_load_4d_elect(dst + c * kChunkBytes, m, bar, c * 64, row0, h, b);
}

// D[tmem] (+)= A·Bᵀ, A and B both [128 × D] K-major tiles (contraction over d)
template <int D>
__device__ __forceinline__ void mma_rows_x_rows(uint32_t d_tmem, const uint8_t* a, const uint8_t* b, bool accum_first) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
  const uint32_t sa = ptx::smem_u32(a), sb = ptx::smem_u32(b);
#pragma unroll
  for (int ks = 0; ks < Cfg<D>::KSTEPS; ++ks) {
    const uint32_t off = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
    ptx::mma_bf16_ss_elect(d_tmem, ptx::sdesc_kmajor(sa + off), ptx::sdesc_kmajor(sb + off), idesc,
                     (accum_first || ks > 0) ? 1u : 0u);
  }
}

__device__ __forceinline__ void ld_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld32(taddr, r);
  ptx::tmem_wait_ld();
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
}

// the math warps' arrive on a barrier counted per warp (count = 4)
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(bar);
}
__device__ __forceinline__ void warp_arrive_addr(uint32_t bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) ptx::mbar_arrive_addr(bar);
}

// compact per-block flags flags[0..n) into an increasing index list (one math warp)
// A block list: the compacted table entries, or — in the unmasked mode (table == nullptr, SURVEY §8f
// NEXT-2, the paper's variant without block masking P:L398, L1073) — every visible block base, base+1, …
struct BlockList {
  const int32_t* idx;
  int base;
  __device__ __forceinline__ int operator[](int k) const { return idx ? __ldg(idx + k) : base + k; }
};

__device__ __forceinline__ int compact_flags(const uint8_t* flags, int n, int32_t* out) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int base = 0; base < n; base += 32) {
    const int j = base + lane;
    const bool f = j < n && flags[j];
    const uint32_t m = __ballot_sync(0xffffffffu, f);
    if (f) out[cnt + __popc(m & ((1u << lane) - 1u))] = j;
    cnt += __popc(m);
  }
  return cnt;
}

}  // namespace sm100
}  // namespace entmax
