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
  for (int c = 0; c < Cfg<D>::KCH; ++c) ptx::tma_load_4d(dst + c * kChunkBytes, m, bar, c * 64, row0, h, b);
}

// D[tmem] (+)= A·Bᵀ, A and B both [128 × D] K-major tiles (contraction over d)
template <int D>
__device__ __forceinline__ void mma_rows_x_rows(uint32_t d_tmem, const uint8_t* a, const uint8_t* b, bool accum_first) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, 128, 0, 0);
  const uint32_t sa = ptx::smem_u32(a), sb = ptx::smem_u32(b);
#pragma unroll
  for (int ks = 0; ks < Cfg<D>::KSTEPS; ++ks) {
    const uint32_t off = (ks >> 2) * kChunkBytes + (ks & 3) * 32;
    ptx::mma_bf16_ss(d_tmem, ptx::sdesc_kmajor(sa + off), ptx::sdesc_kmajor(sb + off), idesc,
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
    ptx::mma_bf16_ss(d_tmem, ptx::sdesc_kmajor(sa + aoff), ptx::sdesc_mnmajor(sb + boff, kChunkBytes), idesc,
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

// =====================================================================================
// K2: output pass (Alg. 2 over the candidate blocks): S → P = [x]_+^e, U = [x]_+^{e−1};
// O += P·V_j, O2 += U·V_j (TRAIN); exact M_ij = any(x > 0); mask row and 𝒬_i table.
// =====================================================================================
template <int D, int E, bool TRAIN>
__global__ void __launch_bounds__(kThreads, 1)
out_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
           const __grid_constant__ CUtensorMap tv, Geom g, AlphaParams ap, const float* __restrict__ tau,
           const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_idx, __nv_bfloat16* __restrict__ o,
           float* __restrict__ o2, uint8_t* __restrict__ mask, int32_t* __restrict__ row_cnt,
           int32_t* __restrict__ row_idx) {
  using C = Cfg<D>;
  constexpr int NST = (D == 64) ? 3 : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::TILE;                  // NST × [K tile | V tile]
  uint8_t* sP = sKV + NST * 2 * C::TILE;        // [128 × 128] bf16
  uint8_t* sU = sP + 32768;                     // [128 × 128] bf16
  uint8_t* aflag = sU + 32768;                  // [Tc]
  __shared__ __align__(8) uint64_t bar_q, kv_full[NST], kv_empty[NST], s_full[2], s_empty[2], p_full, p_empty, o_full;
  __shared__ uint32_t tmem_base_sh;

  const int i = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long li = (long long)bh * g.Tr + i;
  const int ncand = cand_cnt[li];
  const int32_t* list = cand_idx + li * g.Tc;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], 4);
    }
    ptx::mbar_init(&p_full, 4);
    ptx::mbar_init(&p_empty, 1);
    ptx::mbar_init(&o_full, 1);
    ptx::fence_mbar_init();
  }
  for (int j = threadIdx.x; j < g.Tc; j += blockDim.x) aflag[j] = 0;
  if (warp == 5) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_o = tmem + 256, t_o2 = tmem + 256 + D;

  if (warp == 4) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tq);
      ptx::tma_prefetch_desc(&tk);
      ptx::tma_prefetch_desc(&tv);
      ptx::mbar_arrive_expect_tx(&bar_q, C::TILE);
      tma_tile<D>(sQ, &tq, &bar_q, i * kBr, h, b);
      for (int k = 0; k < ncand; ++k) {
        const int j = list[k], st = k % NST;
        ptx::mbar_wait(&kv_empty[st], ((k / NST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * C::TILE);
        tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], j * kBc, h, b);
        tma_tile<D>(sKV + st * 2 * C::TILE + C::TILE, &tv, &kv_full[st], j * kBc, h, b);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      ptx::mbar_wait(&bar_q, 0);
      auto issue_s = [&](int k) {
        const int st = k % NST, sb = k & 1;
        ptx::mbar_wait(&kv_full[st], (k / NST) & 1);
        ptx::mbar_wait(&s_empty[sb], ((k >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        mma_rows_x_rows<D>(tmem + sb * 128, sQ, sKV + st * 2 * C::TILE, false);
        ptx::mma_commit(&s_full[sb]);
      };
      if (ncand > 0) issue_s(0);
      for (int k = 0; k < ncand; ++k) {
        if (k + 1 < ncand) issue_s(k + 1);
        const int st = k % NST;
        ptx::mbar_wait(&p_full, k & 1);
        ptx::tc_fence_after();
        const uint8_t* sV = sKV + st * 2 * C::TILE + C::TILE;
        mma_p_x_tile<D>(t_o, sP, sV, k > 0);
        if (TRAIN) mma_p_x_tile<D>(t_o2, sU, sV, k > 0);
        ptx::mma_commit(&kv_empty[st]);
        ptx::mma_commit(&p_empty);
      }
      ptx::mma_commit(&o_full);
    }
  } else {
    const int row = i * kBr + threadIdx.x;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const float tr = valid ? tau[(long long)bh * g.N + row] : INFINITY;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float usum = 0.f;
    for (int k = 0; k < ncand; ++k) {
      const int j = list[k], sb = k & 1;
      const bool masked = (j + 1) * kBc - 1 > cta_last;
      ptx::mbar_wait(&s_full[sb], (k >> 1) & 1);
      ptx::tc_fence_after();
      ptx::mbar_wait(&p_empty, (k & 1) ^ 1);
      float xmax = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float s[32], p[32], u[32];
        ld_chunk(tmem + lane_base + sb * 128 + c * 32, s);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float x = fmaf(s[e], ap.cp, -tr);
          if (masked && j * kBc + c * 32 + e > my_last) x = -INFINITY;
          xmax = fmaxf(xmax, x);
          p_and_u<E>(x, ap, p[e], u[e]);
          usum += u[e];
        }
        st_row32_bf16(sP, threadIdx.x, c, p);
        if (TRAIN) st_row32_bf16(sU, threadIdx.x, c, u);
      }
      ptx::tc_fence_before();
      warp_arrive(&s_empty[sb]);
      ptx::fence_proxy_async_smem();
      warp_arrive(&p_full);
      if (__any_sync(0xffffffffu, xmax > 0.f) && lane == 0) aflag[j] = 1;
    }
    // epilogue: O, O2 rows from TMEM
    if (ncand > 0) {
      ptx::mbar_wait(&o_full, 0);
      ptx::tc_fence_after();
    }
    const float inv = 1.0f / usum;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      float v[32];
      if (ncand > 0) {
        ld_chunk(tmem + lane_base + 256 + c * 32, v);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.f;
      }
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(o + g.head_off(bh) + (long long)row * g.sn + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(ptx::pack_bf16(v[8 * q], v[8 * q + 1]), ptx::pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                              ptx::pack_bf16(v[8 * q + 4], v[8 * q + 5]), ptx::pack_bf16(v[8 * q + 6], v[8 * q + 7]));
      }
      if (TRAIN) {
        if (ncand > 0) {
          ld_chunk(tmem + lane_base + 256 + D + c * 32, v);
        }
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(o2 + ((long long)bh * g.N + row) * D + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(v[4 * q] * inv, v[4 * q + 1] * inv, v[4 * q + 2] * inv, v[4 * q + 3] * inv);
        }
      }
    }
    ptx::named_bar_sync(1, kMathThreads);
    uint8_t* mrow = mask + li * g.Tc;
    for (int j = threadIdx.x; j < g.Tc; j += kMathThreads) mrow[j] = aflag[j];
    if (warp == 0) {
      const int cnt = compact_flags(aflag, g.Tc, row_idx + li * g.Tc);
      if (lane == 0) row_cnt[li] = cnt;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) ptx::tmem_dealloc<512>(tmem);
}

// =====================================================================================
// K3: dK_j, dV_j over 𝒦_j (Alg. 4).  TMEM lanes = the 128 keys of block j.
//   Sᵀ = K_j Q_iᵀ, dPᵀ = V_j dO_iᵀ; Pᵀ, dSᵀ = Uᵀ ⊙ (dPᵀ − δ_i);
//   dV_j += Pᵀ dO_i, dK_j += dSᵀ Q_i; dK scaled by c at the end (Eq. 1).
// =====================================================================================
template <int D, int E>
__global__ void __launch_bounds__(kThreads, 1)
dkdv_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
            const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g, AlphaParams ap,
            const float* __restrict__ tau, const float* __restrict__ delta, const int32_t* __restrict__ col_cnt,
            const int32_t* __restrict__ col_idx, __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv) {
  using C = Cfg<D>;
  constexpr int NST = (D == 64) ? 2 : 1;
  constexpr uint32_t STAGE = 2 * C::TILE + 1024;   // Q_i | dO_i | τ_i[128] | δ_i[128]
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sStage = sV + C::TILE;
  uint8_t* sPt = sStage + NST * STAGE;
  uint8_t* sDSt = sPt + 32768;
  __shared__ __align__(8) uint64_t bar_kv, qd_full[NST], qd_empty[NST], s_full, s_empty, p_full, p_empty, acc_full;
  __shared__ uint32_t tmem_base_sh;

  const int j = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lj = (long long)bh * g.Tc + j;
  const int cnt = col_cnt[lj];
  const int32_t* list = col_idx + lj * g.Tr;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_kv, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    ptx::mbar_init(&s_full, 1);
    ptx::mbar_init(&s_empty, 4);
    ptx::mbar_init(&p_full, 4);
    ptx::mbar_init(&p_empty, 1);
    ptx::mbar_init(&acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + D;

  if (warp == 4) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tq);
      ptx::tma_prefetch_desc(&tdo);
      ptx::mbar_arrive_expect_tx(&bar_kv, 2 * C::TILE);
      tma_tile<D>(sK, &tk, &bar_kv, j * kBc, h, b);
      tma_tile<D>(sV, &tv, &bar_kv, j * kBc, h, b);
    }
    for (int k = 0; k < cnt; ++k) {
      const int ib = list[k], st = k % NST;
      uint8_t* stg = sStage + st * STAGE;
      ptx::mbar_wait(&qd_empty[st], ((k / NST) & 1) ^ 1);
      float* tq_s = reinterpret_cast<float*>(stg + 2 * C::TILE);
      float* dl_s = tq_s + 128;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = ib * kBr + lane * 4 + e;
        tq_s[lane * 4 + e] = r < g.N ? tau[(long long)bh * g.N + r] : INFINITY;
        dl_s[lane * 4 + e] = r < g.N ? delta[(long long)bh * g.N + r] : 0.f;
      }
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&qd_full[st], 2 * C::TILE);
        tma_tile<D>(stg, &tq, &qd_full[st], ib * kBr, h, b);
        tma_tile<D>(stg + C::TILE, &tdo, &qd_full[st], ib * kBr, h, b);
      }
      __syncwarp();
    }
  } else if (warp == 5) {
    if (lane == 0) {
      ptx::mbar_wait(&bar_kv, 0);
      for (int k = 0; k < cnt; ++k) {
        const int st = k % NST;
        uint8_t* stg = sStage + st * STAGE;
        ptx::mbar_wait(&qd_full[st], (k / NST) & 1);
        ptx::mbar_wait(&s_empty, (k & 1) ^ 1);
        ptx::tc_fence_after();
        mma_rows_x_rows<D>(t_s, sK, stg, false);             // Sᵀ  = K_j Q_iᵀ
        mma_rows_x_rows<D>(t_dp, sV, stg + C::TILE, false);  // dPᵀ = V_j dO_iᵀ
        ptx::mma_commit(&s_full);
        ptx::mbar_wait(&p_full, k & 1);
        ptx::tc_fence_after();
        mma_p_x_tile<D>(t_dv, sPt, stg + C::TILE, k > 0);    // dV += Pᵀ dO_i
        mma_p_x_tile<D>(t_dk, sDSt, stg, k > 0);             // dK += dSᵀ Q_i
        ptx::mma_commit(&qd_empty[st]);
        ptx::mma_commit(&p_empty);
      }
      ptx::mma_commit(&acc_full);
    }
  } else {
    const int key = j * kBc + threadIdx.x;
    const bool valid = key < g.N;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int k = 0; k < cnt; ++k) {
      const int ib = list[k], st = k % NST;
      const uint8_t* stg = sStage + st * STAGE;
      const float* tq_s = reinterpret_cast<const float*>(stg + 2 * C::TILE);
      const float* dl_s = tq_s + 128;
      const bool diag = g.causal && ib == j;   // queries below the key inside the diagonal block
      ptx::mbar_wait(&qd_full[st], (k / NST) & 1);   // τ_i, δ_i staged by the producer warp
      ptx::mbar_wait(&s_full, k & 1);
      ptx::tc_fence_after();
      ptx::mbar_wait(&p_empty, (k & 1) ^ 1);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float s[32], dp[32], p[32], ds[32];
        ld_chunk(lane_base + t_s + c * 32, s);
        ld_chunk(lane_base + t_dp + c * 32, dp);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int ql = c * 32 + e;
          float x = fmaf(s[e], ap.cp, -tq_s[ql]);
          if (!valid || (diag && ql < (int)threadIdx.x)) x = -INFINITY;
          float u;
          p_and_u<E>(x, ap, p[e], u);
          ds[e] = u * (dp[e] - dl_s[ql]);
        }
        st_row32_bf16(sPt, threadIdx.x, c, p);
        st_row32_bf16(sDSt, threadIdx.x, c, ds);
      }
      ptx::tc_fence_before();
      warp_arrive(&s_empty);
      ptx::fence_proxy_async_smem();
      warp_arrive(&p_full);
    }
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
    }
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      float vv[32], kk[32];
      if (cnt > 0) {
        ld_chunk(lane_base + t_dv + c * 32, vv);
        ld_chunk(lane_base + t_dk + c * 32, kk);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) vv[e] = kk[e] = 0.f;
      }
      if (valid) {
        const long long off = g.head_off(bh) + (long long)key * g.sn + c * 32;
        uint4* pv = reinterpret_cast<uint4*>(dv + off);
        uint4* pk = reinterpret_cast<uint4*>(dk + off);
        const float sc = ap.scale;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          pv[q] = make_uint4(ptx::pack_bf16(vv[8 * q], vv[8 * q + 1]), ptx::pack_bf16(vv[8 * q + 2], vv[8 * q + 3]),
                             ptx::pack_bf16(vv[8 * q + 4], vv[8 * q + 5]), ptx::pack_bf16(vv[8 * q + 6], vv[8 * q + 7]));
          pk[q] = make_uint4(ptx::pack_bf16(kk[8 * q] * sc, kk[8 * q + 1] * sc),
                             ptx::pack_bf16(kk[8 * q + 2] * sc, kk[8 * q + 3] * sc),
                             ptx::pack_bf16(kk[8 * q + 4] * sc, kk[8 * q + 5] * sc),
                             ptx::pack_bf16(kk[8 * q + 6] * sc, kk[8 * q + 7] * sc));
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) ptx::tmem_dealloc<512>(tmem);
}

// =====================================================================================
// K4: dQ_i over 𝒬_i (Alg. 5).  S = Q_i K_jᵀ, dP = dO_i V_jᵀ, dS = U ⊙ (dP − δ);
//   dQ_i += dS K_j; dQ scaled by c at the end (Eq. 1).
// =====================================================================================
template <int D, int E>
__global__ void __launch_bounds__(kThreads, 1)
dq_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
          const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g, AlphaParams ap,
          const float* __restrict__ tau, const float* __restrict__ delta, const int32_t* __restrict__ row_cnt,
          const int32_t* __restrict__ row_idx, __nv_bfloat16* __restrict__ dq) {
  using C = Cfg<D>;
  constexpr int NST = (D == 64) ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sDO = sQ + C::TILE;
  uint8_t* sKV = sDO + C::TILE;                 // NST × [K | V]
  uint8_t* sDS = sKV + NST * 2 * C::TILE;     // [128 × 128] bf16
  __shared__ __align__(8) uint64_t bar_q, kv_full[NST], kv_empty[NST], s_full, s_empty, p_full, p_empty, acc_full;
  __shared__ uint32_t tmem_base_sh;

  const int i = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long li = (long long)bh * g.Tr + i;
  const int cnt = row_cnt[li];
  const int32_t* list = row_idx + li * g.Tc;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::mbar_init(&s_full, 1);
    ptx::mbar_init(&s_empty, 4);
    ptx::mbar_init(&p_full, 4);
    ptx::mbar_init(&p_empty, 1);
    ptx::mbar_init(&acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256;

  if (warp == 4) {
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tk);
      ptx::tma_prefetch_desc(&tv);
      ptx::mbar_arrive_expect_tx(&bar_q, 2 * C::TILE);
      tma_tile<D>(sQ, &tq, &bar_q, i * kBr, h, b);
      tma_tile<D>(sDO, &tdo, &bar_q, i * kBr, h, b);
      for (int k = 0; k < cnt; ++k) {
        const int jb = list[k], st = k % NST;
        ptx::mbar_wait(&kv_empty[st], ((k / NST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * C::TILE);
        tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], jb * kBc, h, b);
        tma_tile<D>(sKV + st * 2 * C::TILE + C::TILE, &tv, &kv_full[st], jb * kBc, h, b);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      ptx::mbar_wait(&bar_q, 0);
      for (int k = 0; k < cnt; ++k) {
        const int st = k % NST;
        const uint8_t* sK = sKV + st * 2 * C::TILE;
        ptx::mbar_wait(&kv_full[st], (k / NST) & 1);
        ptx::mbar_wait(&s_empty, (k & 1) ^ 1);
        ptx::tc_fence_after();
        mma_rows_x_rows<D>(t_s, sQ, sK, false);              // S  = Q_i K_jᵀ
        mma_rows_x_rows<D>(t_dp, sDO, sK + C::TILE, false);  // dP = dO_i V_jᵀ
        ptx::mma_commit(&s_full);
        ptx::mbar_wait(&p_full, k & 1);
        ptx::tc_fence_after();
        mma_p_x_tile<D>(t_dq, sDS, sK, k > 0);               // dQ += dS K_j
        ptx::mma_commit(&kv_empty[st]);
        ptx::mma_commit(&p_empty);
      }
      ptx::mma_commit(&acc_full);
    }
  } else {
    const int row = i * kBr + threadIdx.x;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const float tr = valid ? tau[(long long)bh * g.N + row] : INFINITY;
    const float dl = valid ? delta[(long long)bh * g.N + row] : 0.f;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int k = 0; k < cnt; ++k) {
      const int jb = list[k];
      const bool masked = (jb + 1) * kBc - 1 > cta_last;
      ptx::mbar_wait(&s_full, k & 1);
      ptx::tc_fence_after();
      ptx::mbar_wait(&p_empty, (k & 1) ^ 1);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float s[32], dp[32], ds[32];
        ld_chunk(lane_base + t_s + c * 32, s);
        ld_chunk(lane_base + t_dp + c * 32, dp);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float x = fmaf(s[e], ap.cp, -tr);
          if (masked && jb * kBc + c * 32 + e > my_last) x = -INFINITY;
          float p, u;
          p_and_u<E>(x, ap, p, u);
          ds[e] = u * (dp[e] - dl);
        }
        st_row32_bf16(sDS, threadIdx.x, c, ds);
      }
      ptx::tc_fence_before();
      warp_arrive(&s_empty);
      ptx::fence_proxy_async_smem();
      warp_arrive(&p_full);
    }
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
    }
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      float v[32];
      if (cnt > 0) {
        ld_chunk(lane_base + t_dq + c * 32, v);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.f;
      }
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(dq + g.head_off(bh) + (long long)row * g.sn + c * 32);
        const float sc = ap.scale;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(ptx::pack_bf16(v[8 * q] * sc, v[8 * q + 1] * sc),
                              ptx::pack_bf16(v[8 * q + 2] * sc, v[8 * q + 3] * sc),
                              ptx::pack_bf16(v[8 * q + 4] * sc, v[8 * q + 5] * sc),
                              ptx::pack_bf16(v[8 * q + 6] * sc, v[8 * q + 7] * sc));
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace sm100
}  // namespace entmax
