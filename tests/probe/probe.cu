// probe.cu — primitive-level hardware test of the tcgen05 / TMEM / TMA wrappers (test-only library).
//   mode 0: D[128×128] = A[128×K] · B[128×K]ᵀ   (A, B K-major via TMA, K ∈ {64, 128})
//   mode 1: D[128×Nd]  = P[128×128] · V[128×Nd]  (P written by threads into the SW128 layout,
//                                                  V MN-major via TMA, Nd ∈ {64, 128})
#include <cuda_bf16.h>

#include "sm100_ptx.cuh"
#include "tmap.h"

using namespace entmax;

__global__ void __launch_bounds__(128, 1)
probe_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const __nv_bfloat16* P,
             float* D, int mode, int K, int Nd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = smem;              // 32 KB
  uint8_t* sb = smem + 32768;      // 32 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_tma, 1);
    ptx::mbar_init(&bar_mma, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<256>(&tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (mode == 2) {
    // thread r writes row r of A (K bf16 = K/2 packed columns) into TMEM columns 256 + [0, K/2)
    const int r = threadIdx.x;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t w[16];
      for (int e = 0; e < 16; ++e) {
        const __nv_bfloat16* src = P + r * K + (c0 + e) * 2;
        w[e] = ptx::pack_bf16(__bfloat162float(src[0]), __bfloat162float(src[1]));
      }
      ptx::tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + c0, w);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    if (threadIdx.x == 0) {
      const int chunks = K / 64;
      ptx::mbar_arrive_expect_tx(&bar_tma, chunks * 16384);
      for (int c = 0; c < chunks; ++c) ptx::tma_load_4d(sb + c * 16384, &tb, &bar_tma, c * 64, 0, 0, 0);
    }
  } else if (mode == 0) {
    if (threadIdx.x == 0) {
      const int chunks = K / 64;
      ptx::mbar_arrive_expect_tx(&bar_tma, chunks * 2 * 16384);
      for (int c = 0; c < chunks; ++c) {
        ptx::tma_load_4d(sa + c * 16384, &ta, &bar_tma, c * 64, 0, 0, 0);
        ptx::tma_load_4d(sb + c * 16384, &tb, &bar_tma, c * 64, 0, 0, 0);
      }
    }
  } else {
    // thread r writes row r of P (128 keys = 2 chunks of 64) in the K-major SW128 layout
    const int r = threadIdx.x;
    for (int c = 0; c < 2; ++c)
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat16* src = P + r * 128 + c * 64 + u * 8;
        uint32_t w[4];
        for (int e = 0; e < 4; ++e) w[e] = ptx::pack_bf16(__bfloat162float(src[2 * e]), __bfloat162float(src[2 * e + 1]));
        ptx::st_shared_v4(ptx::smem_u32(sa + c * 16384) + ptx::sw128_off(r, u), w[0], w[1], w[2], w[3]);
      }
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
      const int chunks = Nd / 64;
      ptx::mbar_arrive_expect_tx(&bar_tma, chunks * 16384);
      for (int c = 0; c < chunks; ++c) ptx::tma_load_4d(sb + c * 16384, &tb, &bar_tma, c * 64, 0, 0, 0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_wait(&bar_tma, 0);
    ptx::tc_fence_after();
    if (mode == 2) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint32_t off = (ks / 4) * 16384 + (ks % 4) * 32;
        ptx::mma_bf16_ts(tmem, tmem + 256 + ks * 8, ptx::sdesc_kmajor(ptx::smem_u32(sb) + off), idesc, ks > 0);
      }
    } else if (mode == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint32_t off = (ks / 4) * 16384 + (ks % 4) * 32;
        ptx::mma_bf16_ss(tmem, ptx::sdesc_kmajor(ptx::smem_u32(sa) + off), ptx::sdesc_kmajor(ptx::smem_u32(sb) + off),
                         idesc, ks > 0);
      }
    } else {
      const uint32_t idesc = ptx::idesc_bf16(128, Nd, 0, 1);
      for (int ks = 0; ks < 128 / 16; ++ks) {
        const uint32_t aoff = (ks / 4) * 16384 + (ks % 4) * 32;
        const uint32_t boff = ks * 2048;
        ptx::mma_bf16_ss(tmem, ptx::sdesc_kmajor(ptx::smem_u32(sa) + aoff),
                         ptx::sdesc_mnmajor(ptx::smem_u32(sb) + boff, 16384), idesc, ks > 0);
      }
    }
    ptx::mma_commit(&bar_mma);
  }
  __syncwarp();
  ptx::mbar_wait(&bar_mma, 0);
  ptx::tc_fence_after();
  const int ncols = (mode != 1) ? 128 : Nd;
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    uint32_t v[32];
    ptx::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    ptx::tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[row * ncols + c0 + j] = __uint_as_float(v[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<256>(tmem);
}

extern "C" int probe_run(int mode, const void* A, const void* B, const void* P, float* D, int K, int Nd) {
  CUtensorMap ta, tb;
  if (mode == 0 || mode == 2) {
    if (mode == 0 && !make_tmap_bhnd(&ta, A, 1, 1, 128, K, 128LL * K, 128LL * K, K)) return 10;
    if (mode == 2) ta = CUtensorMap{};
    if (!make_tmap_bhnd(&tb, B, 1, 1, 128, K, 128LL * K, 128LL * K, K)) return 11;
  } else {
    ta = CUtensorMap{};
    if (!make_tmap_bhnd(&tb, B, 1, 1, 128, Nd, 128LL * Nd, 128LL * Nd, Nd)) return 12;
  }
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(ta, tb, (const __nv_bfloat16*)P, D, mode, K, Nd);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}
