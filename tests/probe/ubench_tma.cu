// ubench_tma.cu — TMA streaming-rate microbenchmark with the attention kernels' access pattern
// (diagnostic only).  Grid = heads × 64 CTAs; the 64 CTAs of a "head" stream the same sequence of
// [128 × 64] bf16 tiles (one K block = one 16 KB box) in the same order, as the query-block CTAs of the
// τ / output / dQ kernels do.  An elected producer warp issues TMA into an NST-stage ring; a consumer
// warp either releases each stage at once (MMA = 0) or first issues a 128×128×64 SS MMA on it (MMA = 1).
//   BOXES: 16 KB boxes per stage (1 = K only, 2 = K and V as in the output / dQ kernels)
//   MC:    1 = unicast, 2 = CTA pairs each loading half of every box with .multicast::cluster,
//          3 = CTA pairs each loading only its half of every box (cta_group::2 TMA onto the leader's barrier)
//              consumed by a 2-SM MMA (M = 256, each CTA its half of the N = 128 key rows)
#include <cuda_bf16.h>
#include <cstdio>

#include "sm100_ptx.cuh"
#include "tmap.h"

using namespace entmax;

namespace {

template <int BOXES, int MC, int MMA, int NST>
__global__ void __launch_bounds__(128, 1) tma_rate(const __grid_constant__ CUtensorMap tk, int ntile, int nblk,
                                                   long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;                 // 16 KB (MMA A operand, contents irrelevant)
  uint8_t* sK = smem + 16384;         // NST × BOXES × 16 KB
  __shared__ __align__(8) uint64_t full[NST], empty[NST], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = MC >= 2 ? ptx::cluster_ctarank() : 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], MC == 2 ? 2 : 1);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    if (MC == 3) ptx::tmem_alloc_2sm<256>(&tbase); else ptx::tmem_alloc<256>(&tbase);
  }
  ptx::tc_fence_before();
  if (MC >= 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const int head = blockIdx.x / 64;
  const long long t0 = clock64();
  if (warp == 0) {
    for (int t = 0; t < ntile; ++t) {
      const int st = t % NST;
      ptx::mbar_wait(&empty[st], ((t / NST) & 1) ^ 1);
      if (MC != 3 || rank == 0) ptx::mbar_arrive_expect_tx_elect(&full[st], BOXES * 16384);
      const int row = (head * nblk + (t % nblk)) * 128;
#pragma unroll
      for (int bx = 0; bx < BOXES; ++bx) {
        uint8_t* dst = sK + (st * BOXES + bx) * 16384;
        if (MC == 1)
          ptx::tma_load_4d_elect(dst, &tk, &full[st], 0, row + bx * 64 * 0, bx, 0);
        else if (MC == 3)
          ptx::tma_load_4d_2sm_elect(sK + (st * BOXES + bx) * 8192, &tk, ptx::mapa(ptx::smem_u32(&full[st]), 0), 0,
                                     row + (int)rank * 64, bx, 0);
        else
          ptx::tma_load_4d_mc_elect(dst + rank * 8192, &tk, &full[st], 0, row + (int)rank * 64, bx, 0, 0x3);
      }
    }
  } else if (warp == 1 && MC == 3 && rank == 1) {
    if (MMA) ptx::mbar_wait(&done, 0);
    if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = -1;
  } else if (warp == 1) {
    constexpr uint32_t idesc = ptx::idesc_bf16(MC == 3 ? 256 : 128, 128, 0, 0);
    for (int t = 0; t < ntile; ++t) {
      const int st = t % NST;
      ptx::mbar_wait(&full[st], (t / NST) & 1);
      ptx::tc_fence_after();
      if (MMA && MC == 3) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          ptx::mma2_bf16_ss_elect(tmem + (t & 1) * 128, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + ks * 32),
                                  ptx::sdesc_kmajor(ptx::smem_u32(sK + st * BOXES * 8192) + ks * 32), idesc, ks > 0);
        ptx::mma2_commit_mc_elect(&empty[st], 0x3);
      } else if (MMA) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          ptx::mma_bf16_ss_elect(tmem + (t & 1) * 128, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + ks * 32),
                                 ptx::sdesc_kmajor(ptx::smem_u32(sK + st * BOXES * 16384) + ks * 32), idesc, ks > 0);
        if (MC == 2) ptx::mma_commit_mc_elect(&empty[st], 0x3); else ptx::mma_commit_elect(&empty[st]);
      } else {
        if (MC >= 2) {
          if ((threadIdx.x & 31) == 0) {
            ptx::mbar_arrive(&empty[st]);
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&empty[st]), rank ^ 1u));
          }
          __syncwarp();
        } else {
          if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&empty[st]);
          __syncwarp();
        }
      }
    }
    if (MMA) {
      if (MC == 3) ptx::mma2_commit_mc_elect(&done, 0x3); else ptx::mma_commit_elect(&done);
      ptx::mbar_wait(&done, 0);
    }
    if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  if (MC >= 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 2) {
    if (MC == 3) ptx::tmem_dealloc_2sm<256>(tmem); else ptx::tmem_dealloc<256>(tmem);
  }
}

template <int BOXES, int MC, int MMA>
int run(const void* K, int heads, int nblk, int ntile, long long* cycles, float* ms) {
  constexpr int NST = BOXES == 1 ? 6 : 4;
  CUtensorMap tk;
  // K viewed as [1, BOXES, heads·nblk·128, 64]: box bx of a stage is a different "channel" (K / V)
  if (!make_tmap_bhnd(&tk, K, 1, BOXES, heads * nblk * 128, 64, (long long)BOXES * heads * nblk * 128 * 64,
                      (long long)heads * nblk * 128 * 64, 64, MC >= 2 ? 64 : 128))
    return 10;
  const int smem = 16384 + NST * BOXES * 16384 + 1024;
  auto kern = tma_rate<BOXES, MC, MMA, NST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(heads * 64);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MC >= 2 ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const CUtensorMap)tk, ntile, nblk, cycles);
  cudaEventRecord(b);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaEventElapsedTime(ms, a, b);
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

}  // namespace

// K: bf16 buffer of BOXES · heads · nblk · 128 · 64 elements
extern "C" int tma_rate_run(int boxes, int mc, int mma, const void* K, int heads, int nblk, int ntile,
                            long long* cycles, float* ms) {
#define R(B, M, X) \
  if (boxes == B && mc == M && mma == X) return run<B, M, X>(K, heads, nblk, ntile, cycles, ms);
  R(1, 1, 0) R(1, 1, 1) R(1, 2, 0) R(1, 2, 1) R(2, 1, 0) R(2, 1, 1) R(2, 2, 0) R(2, 2, 1)
  R(1, 3, 0) R(1, 3, 1) R(2, 3, 0) R(2, 3, 1)
#undef R
  return 1;
}
