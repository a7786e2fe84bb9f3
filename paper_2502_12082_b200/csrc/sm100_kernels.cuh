// sm100_kernels.cuh — tcgen05 / TMEM / TMA kernels of the bf16 hot path (sm_100a).
//
// Every kernel is warp-specialised, one CTA per 128-row block of one head (B_r = B_c = 128):
//   warps 0-3 : "math" warps — thread t owns TMEM lane t = row t of the S tile (a query row in
//               the τ / output / dQ kernels, a key row in the dK/dV kernel) and runs the
//               per-element α-entmax arithmetic in fp32 registers;
//   warp  4   : TMA producer (lane 0 issues cp.async.bulk.tensor loads into a stage ring);
//   warp  5   : MMA issuer (lane 0 issues tcgen05.mma, commits completions to mbarriers) and
//               owner of the TMEM allocation.
// Operand tiles are [128 rows × 64 bf16] boxes with the 128-byte swizzle; one such tile is
// used K-major (contraction over d) or MN-major (contraction over rows) by descriptor choice.
// P / U / dS tiles produced by the math warps are written to shared memory in the same
// swizzled K-major layout and consumed by SS MMAs.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace entmax {
namespace sm100 {

constexpr int kThreads = 192;
constexpr int kMathThreads = 128;
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

// D[tmem, 128 × D] (+)= A·B, A = [128 × 128] K-major (thread-written P/U/dS tile, two 64-col
// chunks), B = [128 rows × D] tile used MN-major (contraction over its 128 rows)
template <int D>
__device__ __forceinline__ void mma_p_x_tile(uint32_t d_tmem, const uint8_t* a, const uint8_t* b, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, D, 0, 1);
  const uint32_t sa = ptx::smem_u32(a), sb = ptx::smem_u32(b);
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const uint32_t aoff = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
    const uint32_t boff = ks * 2048;
    ptx::mma_bf16_ss_elect(d_tmem, ptx::sdesc_kmajor(sa + aoff), ptx::sdesc_mnmajor(sb + boff, kChunkBytes), idesc,
                     (accumulate || ks > 0) ? 1u : 0u);
  }
}

// write 32 fp32 values (columns c*32 .. c*32+31 of row r) as bf16 into a [128 × 128] K-major
// SW128 tile (two 64-column chunks)
__device__ __forceinline__ void st_row32_bf16(uint8_t* tile, int r, int c, const float* v) {
  const uint32_t base = ptx::smem_u32(tile) + (c >> 1) * kChunkBytes;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t u = (c & 1) * 4 + q;
    ptx::st_shared_v4(base + ptx::sw128_off(r, u), ptx::pack_bf16(v[8 * q + 0], v[8 * q + 1]),
                      ptx::pack_bf16(v[8 * q + 2], v[8 * q + 3]), ptx::pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                      ptx::pack_bf16(v[8 * q + 6], v[8 * q + 7]));
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
