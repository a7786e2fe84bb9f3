// ubench.cu — microbenchmarks of the tcgen05 MMA issue rate and the TMA tile-load rate
// (one CTA per SM), used to size the kernels' pipelines.  Test/diagnostic only.
#include <cuda_bf16.h>
#include <cstdio>

#include "sm100_ptx.cuh"
#include "tmap.h"

using namespace entmax;

// mode 0: MMA only (operands resident in smem): ntile × (K/16) MMAs of 128×128×16
// mode 1: TMA only: ntile loads of a [128 × kdim] bf16 tile through an NST-stage ring
// mode 2: TMA + MMA pipelined (producer lane + MMA lane), like the τ kernel's pass
template <int NST>
__global__ void __launch_bounds__(128, 1)
ubench(const __grid_constant__ CUtensorMap tk, int mode, int ntile, int kdim, int nrows, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + 32768;
  __shared__ uint64_t full[NST], empty[NST], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<256>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const int kch = kdim / 64;
  const uint32_t tile = 128 * kdim * 2;
  const long long t0 = clock64();
  if (mode == 0) {
    if (threadIdx.x == 32) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int t = 0; t < ntile; ++t) {
        for (int ks = 0; ks < kdim / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          ptx::mma_bf16_ss(tmem + (t & 1) * 128, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + off),
                           ptx::sdesc_kmajor(ptx::smem_u32(sK) + off), idesc, ks > 0);
        }
      }
      ptx::mma_commit(&done);
      ptx::mbar_wait(&done, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 6 || mode == 7) {  // MMA only, B cycles through 4 resident stages (6: SS, 7: SS with A cycling too)
    if (threadIdx.x == 32) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int t = 0; t < ntile; ++t) {
        for (int ks = 0; ks < kdim / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          const uint32_t bst = (uint32_t)(t & 3) * tile;
          const uint32_t ast = mode == 7 ? (uint32_t)((t + 1) & 1) * 16384 : 0u;
          ptx::mma_bf16_ss(tmem + (t & 1) * 128, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + ast + off),
                           ptx::sdesc_kmajor(ptx::smem_u32(sK + bst) + off), idesc, ks > 0);
        }
      }
      ptx::mma_commit(&done);
      ptx::mbar_wait(&done, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 3) {  // MMA only, A from TMEM (TS)
    if (threadIdx.x == 32) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int t = 0; t < ntile; ++t)
        for (int ks = 0; ks < kdim / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          ptx::mma_bf16_ts(tmem + (t & 1) * 64, tmem + 128 + ks * 8, ptx::sdesc_kmajor(ptx::smem_u32(sK) + off), idesc,
                           ks > 0);
        }
      ptx::mma_commit(&done);
      ptx::mbar_wait(&done, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 20) {  // TMA only, [128 x 64] tile as two boxes of 64 interleaved rows ([N/2,128] view)
    if (threadIdx.x == 0) {
      for (int t = 0; t < ntile + NST; ++t) {
        if (t >= NST) ptx::mbar_wait(&full[(t - NST) % NST], ((t - NST) / NST) & 1);
        if (t < ntile) {
          const int st = t % NST;
          ptx::mbar_arrive_expect_tx(&full[st], 16384);
          const int row = (((blockIdx.x * 7 + t) * 128) % nrows) / 2;
          for (int c = 0; c < 2; ++c) ptx::tma_load_4d(sK + st * 16384 + c * 8192, &tk, &full[st], c * 64, row, 0, 0);
        }
      }
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode >= 10) {  // TMA only, tile [128 x 64] split into nbox = mode-10 boxes of 128/nbox rows
    const int nbox = mode - 10, brow = 128 / nbox;
    if (threadIdx.x == 0) {
      for (int t = 0; t < ntile + NST; ++t) {
        if (t >= NST) ptx::mbar_wait(&full[(t - NST) % NST], ((t - NST) / NST) & 1);
        if (t < ntile) {
          const int st = t % NST;
          ptx::mbar_arrive_expect_tx(&full[st], 16384);
          const int row = ((blockIdx.x * 7 + t) * 128) % nrows;
          for (int c = 0; c < nbox; ++c) ptx::tma_load_4d(sK + st * 16384 + c * brow * 128, &tk, &full[st], 0, row + c * brow, 0, 0);
        }
      }
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 40 || mode == 41) {  // TMA only: each stage = 2 tiles of 16 KB from 2 row offsets (mode 41: 4 tiles)
    const int per = mode == 40 ? 2 : 4;
    if (threadIdx.x == 0) {
      for (int t = 0; t < ntile + NST; ++t) {
        if (t >= NST) ptx::mbar_wait(&full[(t - NST) % NST], ((t - NST) / NST) & 1);
        if (t < ntile) {
          const int st = t % NST;
          ptx::mbar_arrive_expect_tx(&full[st], per * 16384);
          for (int c = 0; c < per; ++c) {
            const int row = ((blockIdx.x * 7 + t * per + c * 977) * 128) % nrows;
            ptx::tma_load_4d(sK + st * per * 16384 + c * 16384, &tk, &full[st], 0, row, 0, 0);
          }
        }
      }
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 30 || mode == 31) {  // independent: TMA stream (thread 0) || MMA loop on fixed tiles (thread 32)
    if (threadIdx.x == 0) {
      for (int t = 0; t < ntile + NST; ++t) {
        if (t >= NST) ptx::mbar_wait(&full[(t - NST) % NST], ((t - NST) / NST) & 1);
        if (t < ntile) {
          const int st = t % NST;
          ptx::mbar_arrive_expect_tx(&full[st], tile);
          const int row = ((blockIdx.x * 7 + t) * 128) % nrows;
          for (int c = 0; c < kch; ++c) ptx::tma_load_4d(sK + 32768 + st * tile + c * 16384, &tk, &full[st], c * 64, row, 0, 0);
        }
      }
      cycles[blockIdx.x] = clock64() - t0;
    } else if (threadIdx.x == 32) {
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int t = 0; t < ntile; ++t)
        for (int ks = 0; ks < kdim / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          if (mode == 30)
            ptx::mma_bf16_ss(tmem + (t & 1) * 64, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + off),
                             ptx::sdesc_kmajor(ptx::smem_u32(sK) + off), idesc, ks > 0);
          else
            ptx::mma_bf16_ts(tmem + (t & 1) * 64, tmem + 128 + ks * 8, ptx::sdesc_kmajor(ptx::smem_u32(sK) + off),
                             idesc, ks > 0);
        }
      ptx::mma_commit(&done);
      ptx::mbar_wait(&done, 0);
      cycles[gridDim.x + blockIdx.x] = clock64() - t0;
    }
  } else if (mode == 1) {
    if (threadIdx.x == 0) {
      for (int t = 0; t < ntile + NST; ++t) {
        if (t >= NST) ptx::mbar_wait(&full[(t - NST) % NST], ((t - NST) / NST) & 1);
        if (t < ntile) {
          const int st = t % NST;
          ptx::mbar_arrive_expect_tx(&full[st], tile);
          const int row = ((blockIdx.x * 7 + t) * 128) % nrows;
          for (int c = 0; c < kch; ++c) ptx::tma_load_4d(sK + st * tile + c * 16384, &tk, &full[st], c * 64, row, 0, 0);
        }
      }
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else {
    if (threadIdx.x == 0) {  // producer
      for (int t = 0; t < ntile; ++t) {
        const int st = t % NST;
        ptx::mbar_wait(&empty[st], ((t / NST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&full[st], tile);
        const int row = ((blockIdx.x * 7 + t) * 128) % nrows;
        for (int c = 0; c < kch; ++c) ptx::tma_load_4d(sK + st * tile + c * 16384, &tk, &full[st], c * 64, row, 0, 0);
      }
    } else if (threadIdx.x == 32) {  // MMA (mode 2: A = Q tile in smem, mode 4: A in TMEM)
      const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
      for (int t = 0; t < ntile; ++t) {
        const int st = t % NST;
        ptx::mbar_wait(&full[st], (t / NST) & 1);
        ptx::tc_fence_after();
        for (int ks = 0; ks < (mode == 5 ? 2 : 1) * kdim / 16; ++ks) {   // mode 5: two MMA tiles per loaded tile
          const uint32_t off = ((ks % (kdim / 16)) >> 2) * 16384 + (ks & 3) * 32;
          if (mode == 2 || mode == 5)
            ptx::mma_bf16_ss(tmem + (t & 1) * 64, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + off),
                             ptx::sdesc_kmajor(ptx::smem_u32(sK + st * tile) + off), idesc, ks > 0);
          else
            ptx::mma_bf16_ts(tmem + (t & 1) * 64, tmem + 128 + ks * 8,
                             ptx::sdesc_kmajor(ptx::smem_u32(sK + st * tile) + off), idesc, ks > 0);
        }
        ptx::mma_commit(&empty[st]);
      }
      ptx::mma_commit(&done);
      ptx::mbar_wait(&done, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  }
  __syncthreads();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<256>(tmem);
}

// 2-CTA cluster: each CTA loads half (64 rows) of every 16 KB tile, multicast to both; both run
// the same 4-MMA-per-tile loop.  Empty barriers count one commit from each CTA.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
ubench_mc(const __grid_constant__ CUtensorMap tk, int ntile, int nrows, long long* cycles) {
  constexpr int NST = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + 32768;
  __shared__ uint64_t full[NST], empty[NST], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = ptx::cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 2);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<256>(&tbase);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int t = 0; t < ntile; ++t) {
      const int st = t % NST;
      ptx::mbar_wait(&empty[st], ((t / NST) & 1) ^ 1);
      ptx::mbar_arrive_expect_tx(&full[st], 16384);
      const int row = ((blockIdx.x / 2 * 7 + t) * 128) % nrows;
      ptx::tma_load_4d_mc(sK + st * 16384 + rank * 8192, &tk, &full[st], 0, row + (int)rank * 64, 0, 0, 0x3);
    }
  } else if (threadIdx.x == 32) {
    const uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
    for (int t = 0; t < ntile; ++t) {
      const int st = t % NST;
      ptx::mbar_wait(&full[st], (t / NST) & 1);
      ptx::tc_fence_after();
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t off = (ks & 3) * 32;
        ptx::mma_bf16_ss(tmem + (t & 1) * 128, ptx::sdesc_kmajor(ptx::smem_u32(sQ) + off),
                         ptx::sdesc_kmajor(ptx::smem_u32(sK + st * 16384) + off), idesc, ks > 0);
      }
      ptx::mma_commit_mc(&empty[st], 0x3);
    }
    ptx::mma_commit(&done);
    ptx::mbar_wait(&done, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc<256>(tmem);
}

extern "C" int ubench_mc_run(int grid, int ntile, const void* K, int nrows, long long* cycles) {
  CUtensorMap tk;
  if (!make_tmap_bhnd(&tk, K, 1, 1, nrows, 64, (long long)nrows * 64, (long long)nrows * 64, 64, 64)) return 10;
  const int smem = 32768 + 4 * 16384 + 1024;
  cudaFuncSetAttribute(ubench_mc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ubench_mc<<<grid, 128, smem>>>(tk, ntile, nrows, cycles);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

extern "C" int ubench_run(int mode, int nst, int grid, int ntile, int kdim, const void* K, int nrows, long long* cycles,
                          float* ms) {
  CUtensorMap tk;
  if (mode == 20) {
    if (!make_tmap_bhnd(&tk, K, 1, 1, nrows / 2, 128, (long long)nrows * 64, (long long)nrows * 64, 128, 64)) return 10;
  } else {
    const int box_rows = (mode >= 10 && mode < 20) ? 128 / (mode - 10) : 128;
    if (!make_tmap_bhnd(&tk, K, 1, 1, nrows, kdim, (long long)nrows * kdim, (long long)nrows * kdim, kdim, box_rows))
      return 10;
  }
  const int smem = 32768 + 32768 + nst * 128 * kdim * 2 * ((mode == 41) ? 4 : (mode == 40) ? 2 : 1) + 1024;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
#define L(N)                                                                            \
  if (nst == N) {                                                                       \
    cudaFuncSetAttribute(ubench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    ubench<N><<<grid, 128, smem>>>(tk, mode, ntile, kdim, nrows, cycles);               \
  }
  L(2) L(4) L(8)
#undef L
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  cudaEventElapsedTime(ms, a, b);
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

// TMEM → register read bandwidth: nwarp warps each repeatedly load 32 lanes × (x) columns.
template <int X>
__device__ __forceinline__ uint32_t tld(uint32_t taddr) {
  uint32_t r[32];
  if constexpr (X == 32) {
    ptx::tmem_ld32(taddr, r);
  } else {
    uint32_t q[16];
    ptx::tmem_ld16(taddr, q);
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = q[i];
#pragma unroll
    for (int i = 16; i < 32; ++i) r[i] = 0;
  }
  ptx::tmem_wait_ld();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < X; ++i) acc ^= r[i];
  return acc;
}

template <int X>
__global__ void __launch_bounds__(512, 1) tmem_rd(int iters, long long* cycles, uint32_t* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<512>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) acc += tld<X>(tm + ((it * X + warp * 64) & 511));
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * 16 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tbase);
}

extern "C" int tmem_rd_run(int x, int nwarps, int iters, long long* cycles, uint32_t* sink) {
  if (x == 32) tmem_rd<32><<<148, nwarps * 32>>>(iters, cycles, sink);
  else tmem_rd<16><<<148, nwarps * 32>>>(iters, cycles, sink);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
