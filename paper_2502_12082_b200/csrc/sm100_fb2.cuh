// sm100_fb2.cuh — output pass on CTA pairs with 2-SM MMAs (tcgen05.mma.cta_group::2, sm_100a).
//
// Same computation as out_kernel (Alg. 2 over the candidate blocks, App. B.3: S = Q K_jᵀ → x = c'·s − τ,
// P = [x]_+^e, U = [x]_+^{e−1}; O += P V_j, O⁽²⁾ += U V_j; M_ij = any(x > 0)), but the two query blocks
// i, i+1 of a cluster pair share every K/V tile and every MMA: the even CTA issues M = 256 MMAs whose A
// rows are each CTA's own (Q in shared memory for S, P / U in TMEM for the second GEMMs) and whose B
// columns are split between the pair — each CTA loads and holds only its 64-key half of K_j (K-major,
// SW128) and its d/2-column half of V_j (MN-major: SW64 at d = 64, SW128 at d = 128).  Per SM and per
// 128×128 block of work this halves the TMA bytes and the B-operand shared-memory reads and halves the
// MMA instructions.  The pair visits the union of the two blocks' candidate lists (a block that is not a
// candidate of one CTA gives that CTA's rows x <= 0, i.e. exact zeros, so the outputs are unchanged).
// Barriers: every TMA load of the pair completes on the leader's kv_full; the leader's commits arrive on
// both CTAs' kv_empty / s_full / o_full (multicast); both CTAs' math warps arrive on the leader's p_full.
#pragma once

#include "sm100_fb.cuh"

namespace entmax {
namespace sm100 {

template <int D>
struct Out2Cfg {
  static constexpr uint32_t KHALF = Cfg<D>::KCH * (kChunkBytes / 2);   // 64 keys × D
  static constexpr uint32_t VHALF = 128u * (D / 2) * 2u;                 // 128 keys × D/2
  static constexpr uint32_t STAGE = KHALF + VHALF;
  static constexpr int NST = (D == 64) ? 8 : 4;
  static size_t smem(int Tc) {
    return 1024 + Cfg<D>::TILE + (size_t)NST * STAGE + kFbMath * 4 + 2 * (size_t)Tc + 4 * (size_t)Tc + 16;
  }
};

template <int D, int E, bool TRAIN, bool CU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFbThreads, 1)
out2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk64,
            const __grid_constant__ CUtensorMap tvh, Geom g, AlphaParams ap, const float* __restrict__ tau,
            const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_idx, __nv_bfloat16* __restrict__ o,
            float* __restrict__ o2, uint8_t* __restrict__ mask, int32_t* __restrict__ row_cnt,
            int32_t* __restrict__ row_idx) {
  using C = Cfg<D>;
  using OC = Out2Cfg<D>;
  constexpr int NST = OC::NST;
  constexpr int NSB = (D == 64 || !TRAIN) ? 3 : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::TILE;                                      // NST × [K half | V half]
  float* xch = reinterpret_cast<float*>(sKV + NST * OC::STAGE);     // [256]
  uint8_t* aflag = reinterpret_cast<uint8_t*>(xch + kFbMath);      // [Tc] this CTA's exact active blocks
  uint8_t* uflag = aflag + g.Tc;                                    // [Tc] union of the pair's candidates
  int32_t* ulist = reinterpret_cast<int32_t*>(((uintptr_t)(uflag + g.Tc) + 15) & ~(uintptr_t)15);   // [Tc]
  __shared__ __align__(8) uint64_t bar_q, kv_full[NST], kv_empty[NST], s_full[NSB], p_full[NSB], o_full;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_ucnt;

  // causal: the longest query blocks first (the block scheduler issues low indices first); pairs stay
  // (even = cluster rank 0, odd)
  const int i = g.causal ? (((int)gridDim.x - 2 - ((int)blockIdx.x & ~1)) | ((int)blockIdx.x & 1)) : (int)blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool real_cta = i < g.Tr;
  const long long li = (long long)bh * g.Tr + i;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < NSB; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&p_full[s], 16);   // 8 math warps of each CTA
    }
    ptx::mbar_init(&o_full, 1);
    ptx::fence_mbar_init();
  }
  for (int j = threadIdx.x; j < g.Tc; j += blockDim.x) {
    aflag[j] = 0;
    uflag[j] = 0;
  }
  if (warp == 9) ptx::tmem_alloc_2sm<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  ptx::cluster_sync();   // both CTAs' barriers and TMEM exist before the pair's TMA / MMA target them
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_o = tmem + 128 * NSB, t_o2 = t_o + D;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // the τ kernel's outputs are complete and visible
  const bool dense = mask == nullptr;   // unmasked mode: every visible block, no mask / table output
  const int pair0 = i & ~1;
  int ucnt;
  if (dense) {
    ucnt = g.visible_kblocks(min(pair0 + 1, g.Tr - 1));
  } else {
    // union of the pair's candidate lists (both CTAs build the same increasing list)
    for (int q = 0; q < 2; ++q) {
      const int iq = pair0 + q;
      if (iq >= g.Tr) continue;
      const long long lq = (long long)bh * g.Tr + iq;
      const int n = cand_cnt[lq];
      for (int e = threadIdx.x; e < n; e += blockDim.x) uflag[cand_idx[lq * g.Tc + e]] = 1;
    }
    __syncthreads();
    if (warp == 0) {
      const int n = compact_flags(uflag, g.visible_kblocks(min(pair0 + 1, g.Tr - 1)), ulist);
      if (lane == 0) s_ucnt = n;
    }
    __syncthreads();
    ucnt = s_ucnt;
  }
  auto ublock = [&](int k) { return dense ? k : ulist[k]; };

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer (both CTAs)
    ptx::tma_prefetch_desc(&tq);
    ptx::tma_prefetch_desc(&tk64);
    ptx::tma_prefetch_desc(&tvh);
    if (rank == 0) ptx::mbar_arrive_expect_tx_elect(&bar_q, 2 * C::TILE);
    const uint32_t barq_c = ptx::mapa(ptx::smem_u32(&bar_q), 0);
#pragma unroll
    for (int c = 0; c < C::KCH; ++c) ptx::tma_load_4d_2sm_elect(sQ + c * kChunkBytes, &tq, barq_c, c * 64, i * kBr, h, b);
    for (int k = 0; k < ucnt; ++k) {
      const int j = ublock(k), st = k % NST;
      ptx::mbar_wait(&kv_empty[st], ((k / NST) & 1) ^ 1);
      if (rank == 0) ptx::mbar_arrive_expect_tx_elect(&kv_full[st], 2 * OC::STAGE);
      const uint32_t full_c = ptx::mapa(ptx::smem_u32(&kv_full[st]), 0);
      uint8_t* stg = sKV + st * OC::STAGE;
#pragma unroll
      for (int c = 0; c < C::KCH; ++c)   // this CTA's 64 keys of K_j
        ptx::tma_load_4d_2sm_elect(stg + c * (kChunkBytes / 2), &tk64, full_c, c * 64, j * kBc + (int)rank * 64, h, b);
      // this CTA's d/2 columns of V_j (all 128 keys)
      ptx::tma_load_4d_2sm_elect(stg + OC::KHALF, &tvh, full_c, (int)rank * (D / 2), j * kBc, h, b);
    }
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA only)
    if (rank == 0) {
      ptx::mbar_wait(&bar_q, 0);
      constexpr uint32_t idesc_s = ptx::idesc_bf16(256, 128, 0, 0);
      constexpr uint32_t idesc_o = ptx::idesc_bf16(256, D, 0, 1);
      auto issue_s = [&](int k) {
        const int st = k % NST;
        ptx::mbar_wait(&kv_full[st], (k / NST) & 1);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(sQ), sb = ptx::smem_u32(sKV + st * OC::STAGE);
#pragma unroll
        for (int ks = 0; ks < C::KSTEPS; ++ks)
          ptx::mma2_bf16_ss_elect(tmem + (k % NSB) * 128, ptx::sdesc_kmajor(sa + (ks >> 2) * kChunkBytes + (ks & 3) * 32),
                                  ptx::sdesc_kmajor(sb + (ks >> 2) * (kChunkBytes / 2) + (ks & 3) * 32), idesc_s,
                                  ks > 0 ? 1u : 0u);
        ptx::mma2_commit_mc_elect(&s_full[k % NSB], 0x3);
      };
      // B = this CTA's V half used MN-major: SW64 [128 × 32] at d = 64, SW128 [128 × 64] at d = 128;
      // K-step of 16 keys = 16 rows
      auto vdesc = [&](uint32_t sv, int ks) {
        if constexpr (D == 64) return ptx::sdesc_mnmajor_sw64(sv + ks * 1024);
        else return ptx::sdesc_mnmajor(sv + ks * 2048, kChunkBytes);
      };
      for (int k = 0; k < NSB && k < ucnt; ++k) issue_s(k);
      for (int k = 0; k < ucnt; ++k) {
        const int st = k % NST, sb = k % NSB;
        ptx::mbar_wait_cluster(&p_full[sb], (k / NSB) & 1);
        ptx::tc_fence_after();
        const uint32_t buf = tmem + sb * 128;
        const uint32_t sv = ptx::smem_u32(sKV + st * OC::STAGE + OC::KHALF);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          ptx::mma2_bf16_ts_elect(t_o, buf + 8 * ks + (ks >= 4 ? 32 : 0), vdesc(sv, ks), idesc_o, (k > 0 || ks > 0) ? 1u : 0u);
        if (TRAIN) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            ptx::mma2_bf16_ts_elect(t_o2, buf + 32 + 8 * ks + (ks >= 4 ? 32 : 0), vdesc(sv, ks), idesc_o,
                                    (k > 0 || ks > 0) ? 1u : 0u);
        }
        ptx::mma2_commit_mc_elect(&kv_empty[st], 0x3);
        if (k + NSB < ucnt) issue_s(k + NSB);
      }
      ptx::mma2_commit_mc_elect(&o_full, 0x3);
    }
  } else {
    // ---------------------------------------------------------------- math warps (both CTAs)
    const int tid = threadIdx.x, wg = warp >> 2, r = tid & 127;
    const int row = i * kBr + r;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const float tr = valid ? tau[(long long)bh * g.N + row] : kPadTau;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t pfull_c0 = ptx::mapa(ptx::smem_u32(&p_full[0]), 0);
    float usum = 0.f;
    for (int k = 0; k < ucnt; ++k) {
      const int j = ublock(k), sb = k % NSB;
      const bool masked = (j + 1) * kBc - 1 > cta_last;
      const uint32_t col = lane_base + sb * 128 + wg * 64;
      ptx::mbar_wait(&s_full[sb], (k / NSB) & 1);
      ptx::tc_fence_after();
      float s0[32], s1[32];
      ld32f_nowait(col, s0);
      ld32f_nowait(col + 32, s1);
      ptx::tmem_wait_ld();
      uint32_t pp[32], pu[32];
      float2 su = make_float2(0.f, 0.f);
      float xmax = -INFINITY;
      const float2 cp2 = make_float2(ap.cp, ap.cp), ntr2 = make_float2(-tr, -tr);
      const int key0 = j * kBc + wg * 64;
      auto body = [&](auto masked_c) {
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          float2 x = ffma2(make_float2(e < 32 ? s0[e] : s1[e - 32], e < 32 ? s0[e + 1] : s1[e - 31]), cp2, ntr2);
          if constexpr (decltype(masked_c)::value) {
            if (key0 + e > my_last) x.x = kMaskX;
            if (key0 + e + 1 > my_last) x.y = kMaskX;
          }
          if (E != 1 && E != 2) xmax = fmaxf(xmax, fmaxf(x.x, x.y));
          if constexpr (E == 2 || E == 4) {
            uint32_t pb, ub;
            pu_packed<E>(x, pb, ub);
            if constexpr (CU) {
              su = fadd2(su, bf16x2_to_float2(ub));
            } else if constexpr (E == 2) {
              su = fadd2(su, fadd2(x, fabs2(x)));
            } else {
              const float2 bb = fmul2(fmul2(x, fabs2(x)), fabs2(x));
              su = fadd2(su, fadd2(bb, fabs2(bb)));
            }
            pp[e >> 1] = pb;
            pu[e >> 1] = ub;
          } else {
            float2 p, u;
            p_and_u2<E>(x, ap, p, u);
            const uint32_t ub = ptx::pack_bf16(u.x, u.y);
            if constexpr (CU) su = fadd2(su, bf16x2_to_float2(ub));
            else su = fadd2(su, u);
            pp[e >> 1] = ptx::pack_bf16(p.x, p.y);
            pu[e >> 1] = ub;
          }
        }
      };
      if (masked) body(std::true_type{}); else body(std::false_type{});
      if constexpr ((E == 2 || E == 4) && !CU) su = fmul2(su, make_float2(0.5f, 0.5f));
      usum += su.x + su.y;
      if (E == 1 || E == 2) xmax = su.x + su.y;
      ptx::tmem_st32(col, pp);
      if (TRAIN) ptx::tmem_st32(col + 32, pu);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(pfull_c0 + 8u * (uint32_t)sb);
      if (__any_sync(0xffffffffu, xmax > 0.f) && lane == 0) aflag[j] = 1;
    }
    // epilogue: O and O⁽²⁾ = (Σ U V)/ΣU; each column half written by its warpgroup
    xch[tid] = usum;
    ptx::named_bar_sync(1, kFbMath);
    const float inv = 1.0f / (xch[r] + xch[128 + r]);
    if (ucnt > 0) {
      ptx::mbar_wait(&o_full, 0);
      ptx::tc_fence_after();
    }
    store_row_bf16<D / 2>(lane_base + 128 * NSB + wg * (D / 2), o + g.head_off(bh) + (long long)row * g.sn + wg * (D / 2),
                          1.0f, ucnt == 0, valid);
    if (TRAIN) {
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        float v[32];
        if (ucnt > 0) {
          ld_chunk(lane_base + 128 * NSB + D + wg * (D / 2) + c * 32, v);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        }
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(o2 + ((long long)bh * g.N + row) * D + wg * (D / 2) + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(v[4 * q] * inv, v[4 * q + 1] * inv, v[4 * q + 2] * inv, v[4 * q + 3] * inv);
        }
      }
    }
    if (!dense && real_cta) {
      ptx::named_bar_sync(1, kFbMath);
      uint8_t* mrow = mask + li * g.Tc;
      for (int j = tid; j < g.Tc; j += kFbMath) mrow[j] = aflag[j];
      if (warp == 0) {
        const int cnt = compact_flags(aflag, g.Tc, row_idx + li * g.Tc);
        if (lane == 0) row_cnt[li] = cnt;
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();   // no CTA leaves while the pair's MMAs / TMA may still target it
  if (warp == 9) ptx::tmem_dealloc_2sm<512>(tmem);
}

}  // namespace sm100
}  // namespace entmax
