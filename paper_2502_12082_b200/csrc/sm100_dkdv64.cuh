// sm100_dkdv64.cuh — dK_j, dV_j over 𝒦_j (Alg. 4) at d = 64 with half-block units and
// double-buffered Sᵀ/dPᵀ (sm_100a).
//
// The work unit is half a query block (64 queries): Sᵀ_h = K_j Q_hᵀ and dPᵀ_h = V_j dO_hᵀ are TS-MMAs whose A
// operands (K_j, V_j: 32 TMEM columns each) the math warps copy into TMEM once, so only the 64-query halves
// of Q_i and dO_i are read from shared memory; Sᵀ_h/dPᵀ_h (64 + 64 columns) are double-buffered, so the
// MMA issuer computes unit u+2 into a buffer as soon as every math warp holds unit u in registers — the
// next unit's scores no longer wait for the slowest warp to finish the current unit.  Pᵀ_h and dSᵀ_h
// (32 + 32 columns) feed dV += Pᵀ_h dO_h and dK += dSᵀ_h Q_h (TS, B = the halves used MN-major).
// TMEM: K [0,32) V [32,64) | Sᵀ_0 [64,128) dPᵀ_0 [128,192) | Sᵀ_1 [192,256) dPᵀ_1 [256,320) |
//       Pᵀ [320,352) dSᵀ [352,384) | dV [384,448) dK [448,512).
// Same arithmetic, operands and rounding as dkdv_kernel (the per-element math is the same code path).
#pragma once

#include "sm100_fb.cuh"

namespace entmax {
namespace sm100 {

template <int E, bool CU, int MW>
__global__ void __launch_bounds__(dkdv_threads<MW>(), 1)
dkdv64_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
              const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g,
              AlphaParams ap, const float* __restrict__ td, const int32_t* __restrict__ col_cnt,
              const int32_t* __restrict__ col_idx, float* __restrict__ kbar, __nv_bfloat16* __restrict__ dk,
              __nv_bfloat16* __restrict__ dv) {
  constexpr int D = 64;
  using C = Cfg<D>;
  constexpr int NST = 5;                            // Q/dO/τ/δ stages
  constexpr uint32_t STAGE = 2 * C::TILE + 1024;    // Q_i | dO_i | τ_i[128] | δ_i[128]
  constexpr uint32_t HALF = C::TILE / 2;            // 64 rows of a [128 × 64] SW128 tile
  constexpr float kDS = ((E == 2 || E == 4) && !CU) ? 2.f : 1.f;
  constexpr int kMath = 32 * MW;
  constexpr int SL = MW / 4;      // query-column slices of a unit
  constexpr int CW = 64 / SL;     // query columns per thread per unit
  constexpr int WPR = CW / 2;     // bf16x2 words of Pᵀ / dSᵀ per thread
  constexpr int PROD = MW, MMAW = MW + 1;
  constexpr uint32_t C_K = 0, C_V = 32, C_S = 64, C_DP = 128, C_BUF = 128, C_P = 320, C_DS = 352, C_DV = 384,
                     C_DK = 448;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sStage = sV + C::TILE;
  __shared__ __align__(8) uint64_t bar_kv, kvt_full, qd_full[NST], qd_empty[NST], s_full[2], s_empty[2], p_full,
      p_empty, acc_full;
  __shared__ uint32_t tmem_base_sh;

  const int j = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lj = (long long)bh * g.Tc + j;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_kv, 1);
    ptx::mbar_init(&kvt_full, MW);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], MW);
    }
    ptx::mbar_init(&p_full, MW);
    ptx::mbar_init(&p_empty, 1);
    ptx::mbar_init(&acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == MMAW) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // δ and the 𝒦 tables are complete
  const bool dense = col_idx == nullptr;
  const int i0 = g.causal ? (j * kBc) / kBr : 0;
  const int cnt = dense ? g.Tr - i0 : col_cnt[lj];
  const BlockList list{dense ? nullptr : col_idx + lj * g.Tr, i0};
  const int U = 2 * cnt;   // half-block units

  if (warp == PROD) {
    ptx::tma_prefetch_desc(&tq);
    ptx::tma_prefetch_desc(&tdo);
    ptx::mbar_arrive_expect_tx_elect(&bar_kv, 2 * C::TILE);
    tma_tile<D>(sK, &tk, &bar_kv, j * kBc, h, b);
    tma_tile<D>(sV, &tv, &bar_kv, j * kBc, h, b);
    for (int k = 0; k < cnt; ++k) {
      const int ib = list[k], st = k % NST;
      uint8_t* stg = sStage + st * STAGE;
      ptx::mbar_wait(&qd_empty[st], ((k / NST) & 1) ^ 1);
      ptx::mbar_arrive_expect_tx_elect(&qd_full[st], 2 * C::TILE + 2 * kBr * 4);
      ptx::bulk_load_elect(stg + 2 * C::TILE, td + ((long long)bh * g.Tr + ib) * (2 * kBr), 2 * kBr * 4, &qd_full[st]);
      tma_tile<D>(stg, &tq, &qd_full[st], ib * kBr, h, b);
      tma_tile<D>(stg + C::TILE, &tdo, &qd_full[st], ib * kBr, h, b);
    }
  } else if (warp == MMAW) {
    ptx::mbar_wait(&kvt_full, 0);   // K, V copied into TMEM (the TS A operands)
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 64, 0, 0);
    constexpr uint32_t idesc_g = ptx::idesc_bf16(128, 64, 0, 1);
    auto issue_sdp = [&](int u) {
      const int k = u >> 1, hf = u & 1, st = k % NST;
      if (hf == 0) ptx::mbar_wait(&qd_full[st], (k / NST) & 1);
      ptx::mbar_wait(&s_empty[hf], (k & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t sq = ptx::smem_u32(sStage + st * STAGE) + hf * HALF, sdo = sq + C::TILE;
      const uint32_t ts = tmem + C_S + hf * C_BUF, tdp = tmem + C_DP + hf * C_BUF;
#pragma unroll
      for (int ks = 0; ks < C::KSTEPS; ++ks)   // Sᵀ_h = K_j Q_hᵀ
        ptx::mma_bf16_ts_elect(ts, tmem + C_K + 8 * ks, ptx::sdesc_kmajor(sq + ks * 32), idesc_s, ks > 0 ? 1u : 0u);
#pragma unroll
      for (int ks = 0; ks < C::KSTEPS; ++ks)   // dPᵀ_h = V_j dO_hᵀ
        ptx::mma_bf16_ts_elect(tdp, tmem + C_V + 8 * ks, ptx::sdesc_kmajor(sdo + ks * 32), idesc_s, ks > 0 ? 1u : 0u);
      ptx::mma_commit_elect(&s_full[hf]);
    };
    if (U > 0) issue_sdp(0);
    if (U > 1) issue_sdp(1);
    for (int u = 0; u < U; ++u) {
      const int k = u >> 1, hf = u & 1, st = k % NST;
      if (u + 2 < U) issue_sdp(u + 2);   // as soon as the math warps hold unit u (its buffer is free)
      ptx::mbar_wait(&p_full, u & 1);
      ptx::tc_fence_after();
      const uint32_t sq = ptx::smem_u32(sStage + st * STAGE) + hf * HALF, sdo = sq + C::TILE;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)   // dV += Pᵀ_h dO_h (B = dO_h used MN-major: 16 query rows per k-step)
        ptx::mma_bf16_ts_elect(tmem + C_DV, tmem + C_P + 8 * ks, ptx::sdesc_mnmajor(sdo + ks * 2048, kChunkBytes),
                               idesc_g, (u > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)   // dK += dSᵀ_h Q_h
        ptx::mma_bf16_ts_elect(tmem + C_DK, tmem + C_DS + 8 * ks, ptx::sdesc_mnmajor(sq + ks * 2048, kChunkBytes),
                               idesc_g, (u > 0 || ks > 0) ? 1u : 0u);
      ptx::mma_commit_elect(&p_empty);
      if (hf == 1) ptx::mma_commit_elect(&qd_empty[st]);
    }
    ptx::mma_commit_elect(&acc_full);
  } else {
    const int tid = threadIdx.x, wg = warp >> 2, r = tid & 127;
    const int key = j * kBc + r;
    const bool valid = key < g.N;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // K_j (warpgroup 0) and V_j (warpgroup 1) rows into TMEM: column c = elements 2c, 2c+1 of the row
    ptx::mbar_wait(&bar_kv, 0);
    if (wg < 2) {
      const uint32_t src = ptx::smem_u32(wg == 0 ? sK : sV);
      uint32_t w[32];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = ld_shared_u4(src + ptx::sw128_off(r, u));
        w[4 * u] = v.x;
        w[4 * u + 1] = v.y;
        w[4 * u + 2] = v.z;
        w[4 * u + 3] = v.w;
      }
      ptx::tmem_st32(tmem + lane_base + (wg == 0 ? C_K : C_V), w);
      ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    warp_arrive(&kvt_full);
    for (int u = 0; u < U; ++u) {
      const int k = u >> 1, hf = u & 1, st = k % NST;
      const int ib = list[k];
      const uint8_t* stg = sStage + st * STAGE;
      const int q0 = hf * 64 + wg * CW;                                      // first query column (block-local)
      const uint32_t tq4 = ptx::smem_u32(stg + 2 * C::TILE) + q0 * 4;         // τ_i
      const uint32_t dl4 = tq4 + 512;                                         // δ_i
      const bool diag = g.causal && ib == j;
      if (hf == 0) ptx::mbar_wait(&qd_full[st], (k / NST) & 1);   // τ_i, δ_i staged
      ptx::mbar_wait(&s_full[hf], k & 1);
      ptx::tc_fence_after();
      uint32_t ra[CW], rd[CW];
      if constexpr (CW == 32) {
        ptx::tmem_ld32(tmem + lane_base + C_S + hf * C_BUF + wg * CW, ra);
        ptx::tmem_ld32(tmem + lane_base + C_DP + hf * C_BUF + wg * CW, rd);
      } else {
        ptx::tmem_ld16(tmem + lane_base + C_S + hf * C_BUF + wg * CW, ra);
        ptx::tmem_ld16(tmem + lane_base + C_DP + hf * C_BUF + wg * CW, rd);
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      warp_arrive(&s_empty[hf]);
      uint32_t pp[WPR], pd[WPR];
      auto body = [&](auto masked_c) {
#pragma unroll
        for (int q4 = 0; q4 < CW / 4; ++q4) {
          const float4 t4 = ld_shared_f4(tq4 + q4 * 16), d4 = ld_shared_f4(dl4 + q4 * 16);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int c = q4 * 4 + e;
            const float2 tq2 = e == 0 ? make_float2(-t4.x, -t4.y) : make_float2(-t4.z, -t4.w);
            const float2 dq2 = e == 0 ? make_float2(-d4.x, -d4.y) : make_float2(-d4.z, -d4.w);
            float2 x = ffma2(make_float2(__uint_as_float(ra[c]), __uint_as_float(ra[c + 1])), make_float2(ap.cp, ap.cp),
                             tq2);
            if constexpr (decltype(masked_c)::value) {
              if (!valid || (diag && q0 + c < r)) x.x = kMaskX;
              if (!valid || (diag && q0 + c + 1 < r)) x.y = kMaskX;
            }
            const float2 g2 = fadd2(make_float2(__uint_as_float(rd[c]), __uint_as_float(rd[c + 1])), dq2);
            const int w = c >> 1;
            if constexpr (E == 2 || E == 4) {
              uint32_t pb, ub;
              pu_packed<E>(x, pb, ub);
              pp[w] = pb;
              if constexpr (CU) {   // Û (r9)
                pd[w] = mul_bf16x2(ub, ptx::pack_bf16(g2.x, g2.y));
              } else {   // 2dSᵀ = (2u)·(dPᵀ − δ): exact doubling
                const float2 bb = E == 2 ? x : fmul2(fmul2(x, fabs2(x)), fabs2(x));
                const float2 ds2 = fmul2(fadd2(bb, fabs2(bb)), g2);
                pd[w] = ptx::pack_bf16(ds2.x, ds2.y);
              }
            } else {
              float2 p, uu;
              p_and_u2<E>(x, ap, p, uu);
              pp[w] = ptx::pack_bf16(p.x, p.y);
              if constexpr (CU)
                pd[w] = mul_bf16x2(ptx::pack_bf16(uu.x, uu.y), ptx::pack_bf16(g2.x, g2.y));
              else {
                const float2 ds = fmul2(uu, g2);
                pd[w] = ptx::pack_bf16(ds.x, ds.y);
              }
            }
          }
        }
      };
      if (!valid || diag) body(std::true_type{}); else body(std::false_type{});
      ptx::mbar_wait(&p_empty, (u & 1) ^ 1);   // dV/dK(u−1) have consumed Pᵀ, dSᵀ
      ptx::tc_fence_after();
      if constexpr (WPR == 16) {
        ptx::tmem_st16(tmem + lane_base + C_P + wg * WPR, pp);
        ptx::tmem_st16(tmem + lane_base + C_DS + wg * WPR, pd);
      } else {
        ptx::tmem_st8(tmem + lane_base + C_P + wg * WPR, pp);
        ptx::tmem_st8(tmem + lane_base + C_DS + wg * WPR, pd);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      warp_arrive(&p_full);
    }
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
    }
    constexpr int DS = D / SL;   // dK / dV columns stored per thread
    const long long off = g.head_off(bh) + (long long)(valid ? key : 0) * g.sn + wg * DS;
    store_cols_bf16<DS>(tmem + lane_base + C_DV + wg * DS, dv + off, 1.0f, cnt == 0, valid);
    store_cols_bf16<DS>(tmem + lane_base + C_DK + wg * DS, dk + off, ap.scale / kDS, cnt == 0, valid);
    if (kbar != nullptr) {
      // K̄_j (reading r12), as in dkdv_kernel
      constexpr int UNITS = D / 8, RP = kMath / UNITS;
      const int u = tid % UNITS, rp = tid / UNITS;
      const uint32_t kb0 = ptx::smem_u32(sK) + (uint32_t)(u >> 3) * kChunkBytes;
      float a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = 0.f;
#pragma unroll 4
      for (int rr = rp; rr < 128; rr += RP) {
        const uint4 w = ld_shared_u4(kb0 + ptx::sw128_off(rr, u & 7));
        const float2 f0 = bf16x2_to_float2(w.x), f1 = bf16x2_to_float2(w.y), f2 = bf16x2_to_float2(w.z),
                     f3 = bf16x2_to_float2(w.w);
        a[0] += f0.x; a[1] += f0.y; a[2] += f1.x; a[3] += f1.y;
        a[4] += f2.x; a[5] += f2.y; a[6] += f3.x; a[7] += f3.y;
      }
      float* red = reinterpret_cast<float*>(sStage);   // [RP][D] (the stages are idle now)
#pragma unroll
      for (int e = 0; e < 8; ++e) red[rp * D + u * 8 + e] = a[e];
      ptx::named_bar_sync(1, kMath);
      if (tid < D) {
        float sum = 0.f;
        for (int p = 0; p < RP; ++p) sum += red[p * D + tid];
        kbar[((long long)bh * g.Tc + j) * D + tid] = sum / (float)min(kBc, g.N - j * kBc);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == MMAW) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace sm100
}  // namespace entmax
