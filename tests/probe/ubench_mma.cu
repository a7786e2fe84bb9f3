// ubench_mma.cu — tcgen05 MMA issue-rate microbenchmark (diagnostic only, not part of the library).
// Operands resident in shared memory / TMEM (contents irrelevant, zeroed); one CTA (or CTA pair) per
// SM pair; the MMA warp issues `ntile` tiles back to back with elect.sync and fully unrolled,
// constant descriptor offsets — the issue pattern of the attention kernels.  Reports cycles per tile.
//   mode 0: cta_group::1 SS  M128 N128 K64   (4 instr)   S = Q Kᵀ
//   mode 1: cta_group::1 SS  M128 N256 K64   (4 instr)   two key blocks per instruction
//   mode 2: cta_group::1 TS  M128 N64  K128  (8 instr)   O += P V (A = P in TMEM, B MN-major)
//   mode 3: cta_group::1 SS  M128 N64  K128  (8 instr)   A from smem, B MN-major
//   mode 4: cta_group::2 SS  M256 N128 K64   (4 instr)   CTA pair, leader issues
//   mode 5: cta_group::2 SS  M256 N256 K64   (4 instr)
//   mode 6: cta_group::2 TS  M256 N128 K128  (8 instr)   B MN-major, 64 N-columns per CTA
//   mode 7: cta_group::1 TS  M128 N128 K128  (8 instr)
//   mode 8: cta_group::1 TS  M128 N256 K128  (8 instr)
//   mode 9: cta_group::2 TS  M256 N64  K128  (8 instr)   B MN-major SW64, 32 N-columns per CTA (P·V at d = 64)
//   mode 10: cta_group::2 SS M256 N64  K128  (8 instr)   A K-major SW128, B MN-major SW64
#include <cuda_bf16.h>
#include <cstdio>

#include "sm100_ptx.cuh"

using namespace entmax;

namespace {

__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          ptx::smem_u32(bar)),
      "h"(mask)
      : "memory");
}

template <int MODE>
struct M {
  static constexpr bool pair = MODE == 4 || MODE == 5 || MODE == 6 || MODE == 9 || MODE == 10;
};

template <int MODE>
__device__ __forceinline__ void tile(uint32_t tmem, uint32_t sa, uint32_t sb, int t) {
  constexpr uint32_t CH = 16384;
  if constexpr (MODE == 0) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 128, 0, 0);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      ptx::mma_bf16_ss_elect(tmem + (t & 1) * 128, ptx::sdesc_kmajor(sa + ks * 32), ptx::sdesc_kmajor(sb + ks * 32), id,
                             ks > 0);
  } else if constexpr (MODE == 1) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 256, 0, 0);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      ptx::mma_bf16_ss_elect(tmem + (t & 1) * 256, ptx::sdesc_kmajor(sa + ks * 32), ptx::sdesc_kmajor(sb + ks * 32), id,
                             ks > 0);
  } else if constexpr (MODE == 2) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 64, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      ptx::mma_bf16_ts_elect(tmem + (t & 1) * 64, tmem + 256 + ks * 8, ptx::sdesc_mnmajor(sb + ks * 2048, CH), id,
                             ks > 0);
  } else if constexpr (MODE == 3) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 64, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      ptx::mma_bf16_ss_elect(tmem + (t & 1) * 64, ptx::sdesc_kmajor(sa + (ks >> 2) * CH + (ks & 3) * 32),
                             ptx::sdesc_mnmajor(sb + ks * 2048, CH), id, ks > 0);
  } else if constexpr (MODE == 4) {
    constexpr uint32_t id = ptx::idesc_bf16(256, 128, 0, 0);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      mma2_ss(tmem + (t & 1) * 128, ptx::sdesc_kmajor(sa + ks * 32), ptx::sdesc_kmajor(sb + ks * 32), id, ks > 0);
  } else if constexpr (MODE == 5) {
    constexpr uint32_t id = ptx::idesc_bf16(256, 256, 0, 0);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      mma2_ss(tmem + (t & 1) * 256, ptx::sdesc_kmajor(sa + ks * 32), ptx::sdesc_kmajor(sb + ks * 32), id, ks > 0);
  } else if constexpr (MODE == 6) {
    constexpr uint32_t id = ptx::idesc_bf16(256, 128, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      mma2_ts(tmem + (t & 1) * 128, tmem + 256 + ks * 8, ptx::sdesc_mnmajor(sb + ks * 2048, CH), id, ks > 0);
  } else if constexpr (MODE == 7) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 128, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      ptx::mma_bf16_ts_elect(tmem + (t & 1) * 128, tmem + 256 + ks * 8, ptx::sdesc_mnmajor(sb + ks * 2048, CH), id,
                             ks > 0);
  } else if constexpr (MODE == 9) {
    constexpr uint32_t id = ptx::idesc_bf16(256, 64, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      mma2_ts(tmem + (t & 1) * 64, tmem + 256 + ks * 8, ptx::sdesc_mnmajor_sw64(sb + ks * 1024), id, ks > 0);
  } else if constexpr (MODE == 10) {
    constexpr uint32_t id = ptx::idesc_bf16(256, 64, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      mma2_ss(tmem + (t & 1) * 64, ptx::sdesc_kmajor(sa + (ks >> 2) * CH + (ks & 3) * 32),
              ptx::sdesc_mnmajor_sw64(sb + ks * 1024), id, ks > 0);
  } else if constexpr (MODE == 8) {
    constexpr uint32_t id = ptx::idesc_bf16(128, 256, 0, 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      ptx::mma_bf16_ts_elect(tmem + 0, tmem + 256 + ks * 8, ptx::sdesc_mnmajor(sb + ks * 2048, CH), id, ks > 0);
  }
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_rate(int ntile, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tbase;
  constexpr bool PAIR = M<MODE>::pair;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(ptx::smem_u32(&tbase))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      ptx::tmem_alloc<512>(&tbase);
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  if constexpr (PAIR) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sa = ptx::smem_u32(smem), sb = sa + 32768;
  const bool leader = !PAIR || ptx::cluster_ctarank() == 0;
  if (warp == 0 && leader) {
    const long long t0 = clock64();
#pragma unroll 1
    for (int t = 0; t < ntile; ++t) tile<MODE>(tmem, sa, sb, t);
    if constexpr (PAIR) commit2_mc(&done, 0x3);
    else ptx::mma_commit_elect(&done);
    ptx::mbar_wait(&done, 0);
    if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = clock64() - t0;
  } else if (PAIR && warp == 0) {
    ptx::mbar_wait(&done, 0);
    if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = -1;
  }
  ptx::tc_fence_before();
  if constexpr (PAIR) ptx::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      ptx::tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
int run(int grid, int ntile, long long* cycles, float* ms) {
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mma_rate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = M<MODE>::pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaError_t e = cudaLaunchKernelEx(&cfg, mma_rate<MODE>, ntile, cycles);
  cudaEventRecord(b);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaEventElapsedTime(ms, a, b);
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

}  // namespace

extern "C" int mma_rate_run(int mode, int grid, int ntile, long long* cycles, float* ms) {
  switch (mode) {
    case 0: return run<0>(grid, ntile, cycles, ms);
    case 1: return run<1>(grid, ntile, cycles, ms);
    case 2: return run<2>(grid, ntile, cycles, ms);
    case 3: return run<3>(grid, ntile, cycles, ms);
    case 4: return run<4>(grid, ntile, cycles, ms);
    case 5: return run<5>(grid, ntile, cycles, ms);
    case 6: return run<6>(grid, ntile, cycles, ms);
    case 7: return run<7>(grid, ntile, cycles, ms);
    case 8: return run<8>(grid, ntile, cycles, ms);
    case 9: return run<9>(grid, ntile, cycles, ms);
    case 10: return run<10>(grid, ntile, cycles, ms);
  }
  return 1;
}
