// sm100_dkdv_slc.cuh — dK_j, dV_j over 𝒦_j (Alg. 4) at d = 64 with per-slice handshakes
// (sm_100a).
//
// Same arithmetic, operands and rounding as dkdv_kernel (sm100_fb.cuh); what differs is who waits for
// whom.  dkdv_kernel hands the Sᵀ/dPᵀ tile and the Pᵀ/dSᵀ tile to the MMA warp as wholes, so every tile
// waits for the slowest of the 16 math warps (the warps sharing a scheduler finish a tile up to ~1000
// cycles apart).  Here the 128 query columns of a tile are four slices of 32, one per
// group of four math warps (warp w: TMEM lane quadrant w & 3, slice w >> 2), and each slice is its own
// pipeline:
//   Sᵀ_s = K_j Q_sᵀ, dPᵀ_s = V_j dO_sᵀ   (TS-MMAs, M = 128 keys, N = 32 queries, K = d: the A operands
//                                          K_j, V_j sit in TMEM — copied there once — so the N = 32 MMAs
//                                          read only the 32 query rows from shared memory)
//   math: Pᵀ_s, dSᵀ_s = Uᵀ ⊙ (dPᵀ − δ) written over the slice's own Sᵀ_s / dPᵀ_s columns
//   dV += Pᵀ_s dO_s, dK += dSᵀ_s Q_s      (TS-MMAs over the slice's 32 queries, two k-steps)
// and the next tile's Sᵀ_s/dPᵀ_s are issued right behind that slice's dV/dK MMAs (the in-order tensor
// pipe finishes reading Pᵀ_s, dSᵀ_s before they are overwritten).  A slice's four warps therefore only
// ever wait for each other and for their own MMAs.
// TMEM: K [0,32) V [32,64) | Sᵀ [64,192) (slice s at 64 + 32s, Pᵀ_s over its first 16 columns) |
//       dPᵀ [192,320) (dSᵀ_s over the first 16 of slice s) | dV [320,384) dK [384,448).
#pragma once

#include "sm100_fb.cuh"

namespace entmax {
namespace sm100 {

constexpr int kSlcMW = 16;   // math warps: four slices × four lane quadrants

template <int E, bool CU>
__global__ void __launch_bounds__(dkdv_threads<kSlcMW>(), 1)
dkdv_slc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g,
                AlphaParams ap, const float* __restrict__ td, const int32_t* __restrict__ col_cnt,
                const int32_t* __restrict__ col_idx, float* __restrict__ kbar, __nv_bfloat16* __restrict__ dk,
                __nv_bfloat16* __restrict__ dv) {
  constexpr int D = 64, MW = kSlcMW, NS = 4;
  using C = Cfg<D>;
  constexpr int NST = 5;                           // Q/dO/τ/δ stages
  constexpr uint32_t STAGE = 2 * C::TILE + 1024;   // Q_i | dO_i | τ_i[128] | δ_i[128]
  constexpr float kDS = ((E == 2 || E == 4) && !CU) ? 2.f : 1.f;   // the stored dSᵀ is kDS·dSᵀ (exact doubling)
  constexpr int kMath = 32 * MW;
  constexpr int CW = 128 / NS;   // query columns per slice (32)
  constexpr int WPR = CW / 2;    // bf16x2 words of Pᵀ_s / dSᵀ_s per thread (16)
  constexpr int PROD = MW, MMAW = MW + 1;
  constexpr uint32_t C_K = 0, C_V = 32, C_S = 64, C_DP = 192, C_DV = 320, C_DK = 384;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sStage = sV + C::TILE;
  __shared__ __align__(8) uint64_t bar_kv, kvt_full, qd_full[NST], qd_empty[NST], s_full[NS], p_full[NS], acc_full;
  __shared__ uint32_t tmem_base_sh;

  const int j = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5;
  const long long lj = (long long)bh * g.Tc + j;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_kv, 1);
    ptx::mbar_init(&kvt_full, MW);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&p_full[s], MW / NS);
    }
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
  const bool dense = col_idx == nullptr;   // unmasked mode: every query block that sees key block j
  const int i0 = g.causal ? (j * kBc) / kBr : 0;
  const int cnt = dense ? g.Tr - i0 : col_cnt[lj];
  const BlockList list{dense ? nullptr : col_idx + lj * g.Tr, i0};

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
    ptx::mbar_wait(&kvt_full, 0);   // K_j, V_j copied into TMEM (the A operands of Sᵀ_s, dPᵀ_s)
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, CW, 0, 0);   // N = 32 query rows, K-major
    constexpr uint32_t idesc_g = ptx::idesc_bf16(128, D, 0, 1);    // N = d, B MN-major
    const uint32_t stage0 = ptx::smem_u32(sStage);
    // Sᵀ_s(k) and dPᵀ_s(k): rows 32s .. 32s+31 of the K-major Q_i / dO_i tiles (+4 KB: four SW128 atoms)
    auto issue_sdp = [&](int k, int s) {
      const int st = k % NST;
      if (s == 0) ptx::mbar_wait(&qd_full[st], (k / NST) & 1);
      ptx::tc_fence_after();
      const uint32_t sq = stage0 + st * STAGE + s * (CW * 128), sdo = sq + C::TILE;
#pragma unroll
      for (int ks = 0; ks < C::KSTEPS; ++ks)
        ptx::mma_bf16_ts_elect(tmem + C_S + CW * s, tmem + C_K + 8 * ks, ptx::sdesc_kmajor(sq + ks * 32), idesc_s,
                               ks > 0 ? 1u : 0u);
#pragma unroll
      for (int ks = 0; ks < C::KSTEPS; ++ks)
        ptx::mma_bf16_ts_elect(tmem + C_DP + CW * s, tmem + C_V + 8 * ks, ptx::sdesc_kmajor(sdo + ks * 32), idesc_s,
                               ks > 0 ? 1u : 0u);
      ptx::mma_commit_elect(&s_full[s]);
    };
    if (cnt > 0)
      for (int s = 0; s < NS; ++s) issue_sdp(0, s);
    for (int k = 0; k < cnt; ++k) {
      const int st = k % NST;
      const uint32_t sq = stage0 + st * STAGE, sdo = sq + C::TILE;
#pragma unroll 1
      for (int s = 0; s < NS; ++s) {
        ptx::mbar_wait(&p_full[s], k & 1);
        ptx::tc_fence_after();
        // dV += Pᵀ_s dO_s, dK += dSᵀ_s Q_s: k-steps of 16 queries (B MN-major: 16 rows = 2 KB per k-step)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const uint32_t acc = (k > 0 || s > 0 || kk > 0) ? 1u : 0u;
          ptx::mma_bf16_ts_elect(tmem + C_DV, tmem + C_S + CW * s + 8 * kk,
                                 ptx::sdesc_mnmajor(sdo + (2 * s + kk) * 2048, kChunkBytes), idesc_g, acc);
          ptx::mma_bf16_ts_elect(tmem + C_DK, tmem + C_DP + CW * s + 8 * kk,
                                 ptx::sdesc_mnmajor(sq + (2 * s + kk) * 2048, kChunkBytes), idesc_g, acc);
        }
        if (s == NS - 1) ptx::mma_commit_elect(&qd_empty[st]);   // every MMA reading stage st is issued
        if (k + 1 < cnt) issue_sdp(k + 1, s);
      }
    }
    ptx::mma_commit_elect(&acc_full);
  } else {
    const int tid = threadIdx.x, s = warp >> 2, r = tid & 127;
    const int key = j * kBc + r;
    const bool valid = key < g.N;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // K_j (slice 0's warps) and V_j (slice 1's) rows into TMEM: column c = elements 2c, 2c+1 of the row
    ptx::mbar_wait(&bar_kv, 0);
    if (s < 2) {
      const uint32_t src = ptx::smem_u32(s == 0 ? sK : sV);
      uint32_t w[32];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = ld_shared_u4(src + ptx::sw128_off(r, u));
        w[4 * u] = v.x;
        w[4 * u + 1] = v.y;
        w[4 * u + 2] = v.z;
        w[4 * u + 3] = v.w;
      }
      ptx::tmem_st32(tmem + lane_base + (s == 0 ? C_K : C_V), w);
      ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    warp_arrive(&kvt_full);
    const uint32_t tq_a0 = ptx::smem_u32(sStage) + 2 * C::TILE + s * (CW * 4);   // τ_i of the slice's queries
    const uint32_t qdf_a0 = ptx::smem_u32(qd_full), sfull_a = ptx::smem_u32(&s_full[s]),
                   pfull_a = ptx::smem_u32(&p_full[s]);
    const uint32_t t_s = tmem + lane_base + C_S + CW * s, t_dp = tmem + lane_base + C_DP + CW * s;
    // causal: the list is ascending from i0 = j, so only its first entry can be the diagonal block
    const bool diag0 = g.causal && cnt > 0 && list[0] == j;
    int st = 0;
    uint32_t qph = 0;
    for (int k = 0; k < cnt; ++k) {
      const uint32_t tq4 = tq_a0 + st * STAGE, dl4 = tq4 + 512;
      const bool diag = diag0 && k == 0;   // queries below the key inside the diagonal block
      ptx::mbar_wait_addr(qdf_a0 + 8 * st, qph);   // τ_i, δ_i staged
      if (++st == NST) {
        st = 0;
        qph ^= 1u;
      }
      ptx::mbar_wait_addr(sfull_a, k & 1);
      ptx::tc_fence_after();
      float sv[CW], dpv[CW];
      ld32f_nowait(t_s, sv);
      ld32f_nowait(t_dp, dpv);
      ptx::tmem_wait_ld();
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
            float2 x = ffma2(make_float2(sv[c], sv[c + 1]), make_float2(ap.cp, ap.cp), tq2);
            if constexpr (decltype(masked_c)::value) {
              const int ql = s * CW + c;
              if (!valid || (diag && ql < r)) x.x = kMaskX;
              if (!valid || (diag && ql + 1 < r)) x.y = kMaskX;
            }
            const float2 g2 = fadd2(make_float2(dpv[c], dpv[c + 1]), dq2);
            const int w = c >> 1;
            if constexpr (E == 2 || E == 4) {
              uint32_t pb, ub;
              pu_packed<E>(x, pb, ub);
              pp[w] = pb;
              if constexpr (CU) {   // Û (r9)
                pd[w] = mul_bf16x2(ub, ptx::pack_bf16(g2.x, g2.y));
              } else {   // 2dSᵀ = (2u)·(dPᵀ − δ): exact doubling, no relu (see the dQ kernel)
                const float2 bb = E == 2 ? x : fmul2(fmul2(x, fabs2(x)), fabs2(x));
                const float2 ds2 = fmul2(fadd2(bb, fabs2(bb)), g2);
                pd[w] = ptx::pack_bf16(ds2.x, ds2.y);
              }
            } else {
              float2 p, u;
              p_and_u2<E>(x, ap, p, u);
              pp[w] = ptx::pack_bf16(p.x, p.y);
              if constexpr (CU)   // Û (r9)
                pd[w] = mul_bf16x2(ptx::pack_bf16(u.x, u.y), ptx::pack_bf16(g2.x, g2.y));
              else {
                const float2 ds = fmul2(u, g2);
                pd[w] = ptx::pack_bf16(ds.x, ds.y);
              }
            }
          }
        }
      };
      if (!valid || diag) body(std::true_type{}); else body(std::false_type{});
      // Pᵀ_s, dSᵀ_s over the slice's own Sᵀ_s / dPᵀ_s columns (this warp's loads of them have completed)
      ptx::tmem_st16(t_s, pp);
      ptx::tmem_st16(t_dp, pd);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      warp_arrive_addr(pfull_a);
    }
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
    }
    constexpr int DS = D / NS;   // dK / dV columns stored per thread
    const long long off = g.head_off(bh) + (long long)(valid ? key : 0) * g.sn + s * DS;
    store_cols_bf16<DS>(tmem + lane_base + C_DV + s * DS, dv + off, 1.0f, cnt == 0, valid);
    store_cols_bf16<DS>(tmem + lane_base + C_DK + s * DS, dk + off, ap.scale / kDS, cnt == 0, valid);
    if (kbar != nullptr) {
      // K̄_j = mean of the block's keys (fp32) for the dQ kernel's leak correction (reading r12), as in
      // dkdv_kernel
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
