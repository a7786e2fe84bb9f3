// sm100_fb.cuh — output pass and backward kernels (sm_100a), TMEM-resident P / U / dS.
//
// All three kernels: one CTA per 128-row block of one head, 320 threads —
//   warps 0-7 : math warps.  Warp w owns TMEM lanes 32·(w & 3) (one row per thread) and the
//               column half wg = w >> 2 of every 128-column tile (keys wg·64 .. wg·64+63 in the
//               output / dQ kernels, queries wg·64 .. in the dK/dV kernel);
//   warp  8   : TMA producer (stage ring of operand tiles, mbarrier full/empty);
//   warp  9   : MMA issuer + TMEM owner.
// The math warps write the bf16 operand they produce (P, U, dS, Pᵀ, dSᵀ) straight into TMEM with
// tcgen05.st (two bf16 per 32-bit column: lane = row, column = k/2), and the second GEMM of each
// kernel is a TS-MMA (A from TMEM, B = a [128 × d] tile used MN-major).  Nothing round-trips
// through shared memory, which keeps smem bandwidth for the SS-MMAs and the TMA stream.
#pragma once

#include <type_traits>

#include "sm100_kernels.cuh"
#include "trace.cuh"

namespace entmax {
namespace sm100 {

// CU (consistent Û, reading r9): short rows (N <= kConsistentUMaxN) sum ‖Û‖₁ from the bf16-rounded U
// the U·V MMA sees and form dS = Û ⊙ (dP − δ) from the same rounded Û, so Σ_j dS_ij = 0 holds without
// a 2⁻⁹ mismatch (which does not average out over a 2-3 key support); long rows keep fp32 U.
constexpr int kConsistentUMaxN = 512;
// bf16x2 word → two floats; and a float2 rounded to bf16 (RN) and back
__device__ __forceinline__ float2 bf16x2_to_float2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// dS = Û ⊙ (dP − δ) as one bf16x2 multiply of the two bf16-rounded factors (fp32 product, RN to bf16)
__device__ __forceinline__ uint32_t mul_bf16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// Invisible (causal) keys and padding rows: large finite values instead of ±∞, so the sign-carrying
// power forms (x + |x|, x·|x|, … in pu_packed and the doubled dS) give exact zeros instead of ∞ − ∞.
// Every visible x = c′·s − τ is many orders of magnitude smaller.
constexpr float kMaskX = -1e10f;    // x of an invisible key
constexpr float kPadTau = 1e10f;    // τ of a row past N

constexpr int kFbThreads = 320;
constexpr int kFbMath = 256;

// D[tmem, 128 × D] (+)= A[tmem, 128 × 128 bf16] · B[smem, 128 rows × D, MN-major]
template <int D, typename ACol>
__device__ __forceinline__ void mma_tmem_x_tile(uint32_t d_tmem, ACol acol, const uint8_t* b, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, D, 0, 1);
  const uint32_t sb = ptx::smem_u32(b);
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
    ptx::mma_bf16_ts_elect(d_tmem, acol(ks), ptx::sdesc_mnmajor(sb + ks * 2048, kChunkBytes), idesc,
                     (accumulate || ks > 0) ? 1u : 0u);
}

// dQ leak correction (reading r12): a constant [16 × 128] all-ones bf16 tile (K-major SW128, two 64-column
// chunks of 2 KB; the content is swizzle-invariant) in shared memory, so D_aux[128 × 16] += dS·Onesᵀ gives
// every column of row i the sum ρ_i = Σ_j dŜ_ij of the bf16 dS operand exactly as the dQ MMA accumulates it.
constexpr uint32_t kOnesRows = 16;
constexpr uint32_t kOnesBytes = kOnesRows * 256;
template <typename ACol>
__device__ __forceinline__ void mma_tmem_x_ones(uint32_t d_tmem, ACol acol, const uint8_t* ones, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, kOnesRows, 0, 0);
  const uint32_t so = ptx::smem_u32(ones);
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
    ptx::mma_bf16_ts_elect(d_tmem, acol(ks), ptx::sdesc_kmajor(so + (ks >> 2) * (kOnesRows * 128) + (ks & 3) * 32),
                           idesc, (accumulate || ks > 0) ? 1u : 0u);
}

__device__ __forceinline__ uint4 ld_shared_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr_base_plus_idx16) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr_base_plus_idx16));
  return v;
}

// 32 consecutive columns → 32 floats (no wait)
__device__ __forceinline__ void ld32f_nowait(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  ptx::tmem_ld32(taddr, r);
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
}

// store HALF fp32 columns of one row (TMEM chunk loads) as bf16 × scale to global.  The TMEM loads
// are warp-collective, so every lane loads; only lanes with do_store write.
template <int HALF>
__device__ __forceinline__ void store_row_bf16(uint32_t taddr, __nv_bfloat16* dst, float scale, bool zero,
                                               bool do_store) {
#pragma unroll 1
  for (int c = 0; c < HALF / 32; ++c) {
    float v[32];
    if (!zero) {
      ld_chunk(taddr + c * 32, v);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = 0.f;
    }
    if (!do_store) continue;
    uint4* p = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      p[q] = make_uint4(ptx::pack_bf16(v[8 * q] * scale, v[8 * q + 1] * scale),
                        ptx::pack_bf16(v[8 * q + 2] * scale, v[8 * q + 3] * scale),
                        ptx::pack_bf16(v[8 * q + 4] * scale, v[8 * q + 5] * scale),
                        ptx::pack_bf16(v[8 * q + 6] * scale, v[8 * q + 7] * scale));
  }
}

// Store NC fp32 TMEM columns of one row as bf16 × scale (16-column TMEM loads; warp-collective loads, only
// lanes with do_store write).
template <int NC>
__device__ __forceinline__ void store_cols_bf16(uint32_t taddr, __nv_bfloat16* dst, float scale, bool zero,
                                                bool do_store) {
#pragma unroll 1
  for (int c = 0; c < NC / 16; ++c) {
    uint32_t r[16];
    if (!zero) {
      ptx::tmem_ld16(taddr + c * 16, r);
      ptx::tmem_wait_ld();
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) r[e] = 0u;
    }
    if (!do_store) continue;
    uint4* p = reinterpret_cast<uint4*>(dst + c * 16);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = ptx::pack_bf16(__uint_as_float(r[8 * q + 2 * e]) * scale, __uint_as_float(r[8 * q + 2 * e + 1]) * scale);
      p[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// dQ epilogue with the leak correction (reading r12): row ← c·(acc − ρ·K̄) for NC fp32 columns (16-column
// TMEM loads), K̄ = kb[0..NC) (fp32, global), ρ this row's Σ_j dŜ_ij.
template <int NC>
__device__ __forceinline__ void store_row_bf16_corr(uint32_t taddr, __nv_bfloat16* dst, float scale, bool zero,
                                                    bool do_store, float rho, const float* __restrict__ kb) {
#pragma unroll 1
  for (int c = 0; c < NC / 16; ++c) {
    uint32_t r[16];
    float v[16];
    if (!zero) {
      ptx::tmem_ld16(taddr + c * 16, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = 0.f;
    }
    if (!do_store) continue;
    if (kb != nullptr) {
      const float4* k4 = reinterpret_cast<const float4*>(kb + c * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 kk = __ldg(k4 + q);
        v[4 * q] = fmaf(-rho, kk.x, v[4 * q]);
        v[4 * q + 1] = fmaf(-rho, kk.y, v[4 * q + 1]);
        v[4 * q + 2] = fmaf(-rho, kk.z, v[4 * q + 2]);
        v[4 * q + 3] = fmaf(-rho, kk.w, v[4 * q + 3]);
      }
    }
    uint4* p = reinterpret_cast<uint4*>(dst + c * 16);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      p[q] = make_uint4(ptx::pack_bf16(v[8 * q] * scale, v[8 * q + 1] * scale),
                        ptx::pack_bf16(v[8 * q + 2] * scale, v[8 * q + 3] * scale),
                        ptx::pack_bf16(v[8 * q + 4] * scale, v[8 * q + 5] * scale),
                        ptx::pack_bf16(v[8 * q + 6] * scale, v[8 * q + 7] * scale));
  }
}

// =====================================================================================
// Output pass (Alg. 2 over the candidate blocks, App. B.3): S = Q K_jᵀ → x = c'·s − τ,
// P = [x]_+^e, U = [x]_+^{e−1}; O += P V_j, O⁽²⁾ += U V_j (TRAIN); M_ij = any(x > 0).
// TMEM: NSB S buffers of 128 columns (3 at d = 64, 2 at d = 128 in training) — after the math warps read
// a buffer they overwrite their own 64 columns with P (cols wg·64 + [0,32)) and U (wg·64 + [32,64)) —
// then O and O⁽²⁾.  The MMA issue order S(0) … S(NSB−1) | PV(0) UV(0) S(NSB) | PV(1) UV(1) S(NSB+1) …
// keeps the tensor pipe on later tiles while the math warps work on the current one; S(k+NSB) is issued
// after PV(k) in program order, so the in-order tensor pipe never overwrites P(k) before it is consumed.
// =====================================================================================
template <int MW>
constexpr int out_threads() { return 32 * MW + 64; }

// MW math warps (8 or 16): warp w owns TMEM lanes 32·(w & 3) and the key-column slice w >> 2 of width
// CW = 128·4/MW, whose first CW/4 columns it overwrites with P and the next CW/4 with U.
template <int D, int E, bool TRAIN, bool CU, int MW>
__global__ void __launch_bounds__(out_threads<MW>(), 1)
out_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
           const __grid_constant__ CUtensorMap tv, Geom g, AlphaParams ap, const float* __restrict__ tau,
           const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_idx, __nv_bfloat16* __restrict__ o,
           float* __restrict__ o2, uint8_t* __restrict__ mask, int32_t* __restrict__ row_cnt,
           int32_t* __restrict__ row_idx) {
  using C = Cfg<D>;
  constexpr int NST = (D == 64) ? 6 : 2;    // K/V stages (d = 64: 6 × 32 KB, deep enough to cover the TMA latency)
  // S buffers in TMEM (P/U overwrite their own S buffer): three where the accumulators leave room
  // (d = 64: 3 × 128 + O 64 + O⁽²⁾ 64; inference d = 128: 3 × 128 + O 128), so S(k+3) runs while the math
  // warps still work on tiles k+1 and k+2
  constexpr int NSB = (D == 64 || !TRAIN) ? 3 : 2;
  constexpr int kMath = 32 * MW;
  constexpr int SL = MW / 4;           // key-column slices
  constexpr int CW = 128 / SL;         // key columns per thread
  constexpr int WPR = CW / 2;          // bf16x2 words of P (and of U) per thread
  constexpr int PROD = MW, MMAW = MW + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::TILE;                  // NST × [K tile | V tile]
  float* xch = reinterpret_cast<float*>(sKV + NST * 2 * C::TILE);   // [kMath]
  uint8_t* aflag = reinterpret_cast<uint8_t*>(xch + kMath);         // [Tc]
  __shared__ __align__(8) uint64_t bar_q, kv_full[NST], kv_empty[NST], s_full[NSB], p_full[NSB], o_full;
  __shared__ uint32_t tmem_base_sh;

  // causal: the longest query blocks first (the block scheduler issues low indices first)
  const int i = g.causal ? g.Tr - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long li = (long long)bh * g.Tr + i;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < NSB; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&p_full[s], MW);
    }
    ptx::mbar_init(&o_full, 1);
    ptx::fence_mbar_init();
  }
  for (int j = threadIdx.x; j < g.Tc; j += blockDim.x) aflag[j] = 0;
  if (threadIdx.x == 0) ENTMAX_TRACE_K(1, 8002);
  if (warp == MMAW) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_o = tmem + 128 * NSB, t_o2 = t_o + D;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // the τ kernel's outputs are complete and visible
  const bool dense = mask == nullptr;   // unmasked mode: every visible block, no mask / table output
  const int ncand = dense ? g.visible_kblocks(i) : cand_cnt[li];
  const BlockList list{dense ? nullptr : cand_idx + li * g.Tc, 0};

  if (warp == PROD) {
    ptx::tma_prefetch_desc(&tq);
    ptx::tma_prefetch_desc(&tk);
    ptx::tma_prefetch_desc(&tv);
    ptx::mbar_arrive_expect_tx_elect(&bar_q, C::TILE);
    tma_tile<D>(sQ, &tq, &bar_q, i * kBr, h, b);
    for (int k = 0; k < ncand; ++k) {
      const int j = list[k], st = k % NST;
      ptx::mbar_wait(&kv_empty[st], ((k / NST) & 1) ^ 1);
      ENTMAX_TRACE_K(1, 8 * k + 7);
#ifdef ENTMAX_FB_HALFTMA   // diagnostics: half the streamed bytes (results invalid)
      ptx::mbar_arrive_expect_tx_elect(&kv_full[st], C::TILE);
      tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], j * kBc, h, b);
#else
      ptx::mbar_arrive_expect_tx_elect(&kv_full[st], 2 * C::TILE);
      tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], j * kBc, h, b);
      tma_tile<D>(sKV + st * 2 * C::TILE + C::TILE, &tv, &kv_full[st], j * kBc, h, b);
#endif
    }
  } else if (warp == MMAW) {
    ptx::mbar_wait(&bar_q, 0);
    auto issue_s = [&](int k) {
      const int st = k % NST;
      ptx::mbar_wait(&kv_full[st], (k / NST) & 1);
      ptx::tc_fence_after();
      mma_rows_x_rows<D>(tmem + (k % NSB) * 128, sQ, sKV + st * 2 * C::TILE, false);
      ptx::mma_commit_elect(&s_full[k % NSB]);
      ENTMAX_TRACE_K(1, 8 * k + 0);
    };
    for (int k = 0; k < NSB && k < ncand; ++k) issue_s(k);
    for (int k = 0; k < ncand; ++k) {
      const int st = k % NST, sb = k % NSB;
      ptx::mbar_wait(&p_full[sb], (k / NSB) & 1);
      ENTMAX_TRACE_K(1, 8 * k + 1);
      ptx::tc_fence_after();
      const uint32_t buf = tmem + sb * 128;
      const uint8_t* sV = sKV + st * 2 * C::TILE + C::TILE;
      // k-step ks (16 keys = 8 words) lives in slice ks / KPS: P at its start, U CW/4 columns later
      constexpr int KPS = CW / 16;
      mma_tmem_x_tile<D>(t_o, [&](int ks) { return buf + CW * (ks / KPS) + 8 * (ks % KPS); }, sV, k > 0);
      if (TRAIN)
        mma_tmem_x_tile<D>(t_o2, [&](int ks) { return buf + CW * (ks / KPS) + WPR + 8 * (ks % KPS); }, sV, k > 0);
      ptx::mma_commit_elect(&kv_empty[st]);
      if (k + NSB < ncand) issue_s(k + NSB);
    }
    ptx::mma_commit_elect(&o_full);
  } else {
    const int tid = threadIdx.x, wg = warp >> 2, r = tid & 127;
    const int row = i * kBr + r;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const float tr = valid ? tau[(long long)bh * g.N + row] : kPadTau;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    // barrier addresses as 32-bit shared offsets and the buffer index / phase as running counters (no
    // per-tile generic→shared conversion or division)
    const uint32_t sfull_a0 = ptx::smem_u32(s_full), pfull_a0 = ptx::smem_u32(p_full);
    int sb = 0;
    uint32_t sph = 0;
    float usum = 0.f;
    for (int k = 0; k < ncand; ++k) {
      const int j = list[k];
      const bool masked = (j + 1) * kBc - 1 > cta_last;
      const uint32_t col = lane_base + sb * 128 + wg * CW;
      ptx::mbar_wait_addr(sfull_a0 + 8 * sb, sph);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(1, 8 * k + 3);
      ptx::tc_fence_after();
      float s0[32], s1[32];
      ld32f_nowait(col, s0);
      if constexpr (CW == 64) ld32f_nowait(col + 32, s1);
      ptx::tmem_wait_ld();
      uint32_t pp[WPR], pu[WPR];
      float2 su = make_float2(0.f, 0.f);     // Σ U of this step (> 0 ⟺ some x > 0 for E ∈ {1, 2})
      float xmax = -INFINITY;
      const float2 cp2 = make_float2(ap.cp, ap.cp), ntr2 = make_float2(-tr, -tr);
      const int key0 = j * kBc + wg * CW;
      auto body = [&](auto masked_c) {
#pragma unroll
        for (int e = 0; e < CW; e += 2) {
          float2 x = ffma2(make_float2(e < 32 ? s0[e] : s1[e - 32], e < 32 ? s0[e + 1] : s1[e - 31]), cp2, ntr2);
          if constexpr (decltype(masked_c)::value) {
            if (key0 + e > my_last) x.x = kMaskX;
            if (key0 + e + 1 > my_last) x.y = kMaskX;
          }
          if (E != 1 && E != 2) xmax = fmaxf(xmax, fmaxf(x.x, x.y));
          if constexpr (E == 2 || E == 4) {
            // P̂, Û packed straight from x (pu_packed); ΣU from 2u = x + |x| (E = 2) or b + |b| (E = 4),
            // exact doublings, halved at the end — bitwise the same sums as Σ relu(·)
            uint32_t pb, ub;
            pu_packed<E>(x, pb, ub);
            if constexpr (CU) {
              su = fadd2(su, bf16x2_to_float2(ub));   // ‖Û‖₁ of the rounded U the U·V MMA sees (r9)
            } else if constexpr (E == 2) {
              su = fadd2(su, fadd2(x, fabs2(x)));
            } else {
              const float2 b = fmul2(fmul2(x, fabs2(x)), fabs2(x));
              su = fadd2(su, fadd2(b, fabs2(b)));
            }
            pp[e >> 1] = pb;
            pu[e >> 1] = ub;
          } else {
            float2 p, u;
            p_and_u2<E>(x, ap, p, u);
            // U enters the U·V MMA rounded to bf16 (c14); with CU, ‖U‖₁ is summed from the same rounded
            // values (reading r9)
            const uint32_t ub = ptx::pack_bf16(u.x, u.y);
            if constexpr (CU) su = fadd2(su, bf16x2_to_float2(ub));
            else su = fadd2(su, u);
            pp[e >> 1] = ptx::pack_bf16(p.x, p.y);
            pu[e >> 1] = ub;
          }
        }
      };
#ifdef ENTMAX_FB_NOMATH   // diagnostics: pipeline time without the per-element math (results invalid)
      if (tr == 12345.f)
#endif
      if (masked) body(std::true_type{}); else body(std::false_type{});
      if constexpr ((E == 2 || E == 4) && !CU) su = fmul2(su, make_float2(0.5f, 0.5f));
      usum += su.x + su.y;
      if (E == 1 || E == 2) xmax = su.x + su.y;   // exact: every U > 0 iff x > 0 (no underflow for e <= 2)
      if (threadIdx.x == 0) ENTMAX_TRACE_K(1, 8 * k + 4);
      if constexpr (WPR == 32) {
        ptx::tmem_st32(col, pp);
        if (TRAIN) ptx::tmem_st32(col + 32, pu);
      } else {
        ptx::tmem_st16(col, pp);
        if (TRAIN) ptx::tmem_st16(col + 16, pu);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      warp_arrive_addr(pfull_a0 + 8 * sb);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(1, 8 * k + 6);
      if (__any_sync(0xffffffffu, xmax > 0.f) && lane == 0) aflag[j] = 1;
      if (++sb == NSB) {
        sb = 0;
        sph ^= 1u;
      }
    }
    // epilogue: O and O⁽²⁾ = (Σ U V)/ΣU; each column half written by its warpgroup
    xch[tid] = usum;
    ptx::named_bar_sync(1, kMath);
    float usr = 0.f;
#pragma unroll
    for (int q = 0; q < SL; ++q) usr += xch[q * 128 + r];
    const float inv = 1.0f / usr;
    if (ncand > 0) {
      ptx::mbar_wait(&o_full, 0);
      ptx::tc_fence_after();
    }
    constexpr int DS = D / SL;   // O / O⁽²⁾ columns stored per thread
    store_cols_bf16<DS>(lane_base + 128 * NSB + wg * DS, o + g.head_off(bh) + (long long)row * g.sn + wg * DS, 1.0f,
                        ncand == 0, valid);
    if (TRAIN) {
#pragma unroll 1
      for (int c = 0; c < DS / 16; ++c) {
        uint32_t rv[16];
        if (ncand > 0) {
          ptx::tmem_ld16(lane_base + 128 * NSB + D + wg * DS + c * 16, rv);
          ptx::tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) rv[e] = 0u;
        }
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(o2 + ((long long)bh * g.N + row) * D + wg * DS + c * 16);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_float4(__uint_as_float(rv[4 * q]) * inv, __uint_as_float(rv[4 * q + 1]) * inv,
                                 __uint_as_float(rv[4 * q + 2]) * inv, __uint_as_float(rv[4 * q + 3]) * inv);
        }
      }
    }
    if (!dense) {
      ptx::named_bar_sync(1, kMath);
      uint8_t* mrow = mask + li * g.Tc;
      for (int j = tid; j < g.Tc; j += kMath) mrow[j] = aflag[j];
      if (warp == 0) {
        const int cnt = compact_flags(aflag, g.Tc, row_idx + li * g.Tc);
        if (lane == 0) row_cnt[li] = cnt;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ENTMAX_TRACE_K(1, 8003);
  if (warp == MMAW) ptx::tmem_dealloc<512>(tmem);
}

// =====================================================================================
// dQ_i over 𝒬_i (Alg. 5): S = Q_i K_jᵀ, dP = dO_i V_jᵀ (SS-MMAs); dS = U ⊙ (dP − δ) written to
// TMEM; dQ_i += dS K_j (TS-MMA); dQ scaled by c at the end (Eq. 1).
// TMEM: S [0,128), dP [128,256), dS [256,320) (wg·32 + …), dQ [320, 320+D).
// Issue order S,dP(k+1) | dQ(k): the next tile's scores are computed while the math warps form dS(k).
// MW math warps (8 or 16): warp w owns TMEM lanes 32·(w & 3) and the key-column slice w >> 2 of width
// CW = 128·4/MW.
// =====================================================================================
template <int MW>
constexpr int dq_threads() { return 32 * MW + 64; }

template <int D, int E, bool CU, int MW>
__global__ void __launch_bounds__(dq_threads<MW>(), 1)
dq_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
          const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g, AlphaParams ap,
          const float* __restrict__ tau, const float* __restrict__ delta, const int32_t* __restrict__ row_cnt,
          const int32_t* __restrict__ row_idx, const float* __restrict__ kbar, __nv_bfloat16* __restrict__ dq) {
  using C = Cfg<D>;
  constexpr int NST = (D == 64) ? 5 : 2;   // K/V stages
  constexpr int NDS = (D == 64) ? 2 : 1;
  constexpr float kDS = ((E == 2 || E == 4) && !CU) ? 2.f : 1.f;   // the stored dS is kDS·dS (exact doubling)
  constexpr int kMath = 32 * MW;
  constexpr int SL = MW / 4;           // key-column slices
  constexpr int CW = 128 / SL;         // key columns per thread
  constexpr int NH = CW / 32;
  constexpr int WPR = CW / 2;          // bf16x2 words of dS per thread
  constexpr int PROD = MW, MMAW = MW + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sDO = sQ + C::TILE;
  uint8_t* sKV = sDO + C::TILE;                 // NST × [K | V]
  uint8_t* sOnes = sKV + NST * 2 * C::TILE;     // [16 × 128] bf16 ones (leak correction, r12)
  __shared__ __align__(8) uint64_t bar_q, kv_full[NST], kv_empty[NST], s_full, s_empty, ds_full[NDS], ds_empty[NDS], acc_full;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_first;                       // first tile (list order) with a non-zero dS in this CTA

  // causal: the longest query blocks first (the block scheduler issues low indices first)
  const int i = g.causal ? g.Tr - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long li = (long long)bh * g.Tr + i;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::mbar_init(&s_full, 1);
    ptx::mbar_init(&s_empty, MW);
    for (int s = 0; s < NDS; ++s) {
      ptx::mbar_init(&ds_full[s], MW);
      ptx::mbar_init(&ds_empty[s], 1);
    }
    ptx::mbar_init(&acc_full, 1);
    ptx::fence_mbar_init();
    s_first = INT_MAX;
  }
  for (uint32_t w = threadIdx.x; w < kOnesBytes / 4; w += blockDim.x)
    reinterpret_cast<uint32_t*>(sOnes)[w] = 0x3f803f80u;   // bf16 1.0 pairs
  ptx::fence_proxy_async_smem();                           // visible to the tcgen05.mma operand reads
  if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8002);
  if (warp == MMAW) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  // TMEM: S [0,128), dP [128,256), dS buffers 64 each from 256, dQ (D), ρ aux (16)
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_ds = tmem + 256, t_dq = tmem + 256 + 64 * NDS, t_aux = t_dq + D;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // the dK/dV kernel (and everything before it, incl. K̄) is complete
  const bool dense = row_idx == nullptr;   // unmasked mode: every visible key block
  const int cnt = dense ? g.visible_kblocks(i) : row_cnt[li];
  const BlockList list{dense ? nullptr : row_idx + li * g.Tc, 0};

  if (warp == PROD) {
    ptx::tma_prefetch_desc(&tk);
    ptx::tma_prefetch_desc(&tv);
    ptx::mbar_arrive_expect_tx_elect(&bar_q, 2 * C::TILE);
    tma_tile<D>(sQ, &tq, &bar_q, i * kBr, h, b);
    tma_tile<D>(sDO, &tdo, &bar_q, i * kBr, h, b);
    for (int k = 0; k < cnt; ++k) {
      const int jb = list[k], st = k % NST;
      ptx::mbar_wait(&kv_empty[st], ((k / NST) & 1) ^ 1);
      ENTMAX_TRACE_K(3, 8 * k + 7);
#ifdef ENTMAX_FB_HALFTMA
      ptx::mbar_arrive_expect_tx_elect(&kv_full[st], C::TILE);
      tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], jb * kBc, h, b);
#else
      ptx::mbar_arrive_expect_tx_elect(&kv_full[st], 2 * C::TILE);
      tma_tile<D>(sKV + st * 2 * C::TILE, &tk, &kv_full[st], jb * kBc, h, b);
      tma_tile<D>(sKV + st * 2 * C::TILE + C::TILE, &tv, &kv_full[st], jb * kBc, h, b);
#endif
    }
  } else if (warp == MMAW) {
    ptx::mbar_wait(&bar_q, 0);
    auto issue_sdp = [&](int k) {
      const int st = k % NST;
      const uint8_t* sK = sKV + st * 2 * C::TILE;
      ptx::mbar_wait(&kv_full[st], (k / NST) & 1);
      ptx::mbar_wait(&s_empty, (k & 1) ^ 1);
      ptx::tc_fence_after();
      mma_rows_x_rows<D>(t_s, sQ, sK, false);              // S  = Q_i K_jᵀ
      mma_rows_x_rows<D>(t_dp, sDO, sK + C::TILE, false);  // dP = dO_i V_jᵀ
      ptx::mma_commit_elect(&s_full);
      ENTMAX_TRACE_K(3, 8 * k + 0);
    };
    if (cnt > 0) issue_sdp(0);
    for (int k = 0; k < cnt; ++k) {
      if (k + 1 < cnt) issue_sdp(k + 1);
      const int st = k % NST;
      const int db = k % NDS;
      const uint32_t dsb = t_ds + 64 * db;
      ptx::mbar_wait(&ds_full[db], (k / NDS) & 1);
      ENTMAX_TRACE_K(3, 8 * k + 1);
      ptx::tc_fence_after();
      mma_tmem_x_tile<D>(t_dq, [&](int ks) { return dsb + 8 * ks; }, sKV + st * 2 * C::TILE, k > 0);
      mma_tmem_x_ones(t_aux, [&](int ks) { return dsb + 8 * ks; }, sOnes, k > 0);   // ρ_i (r12)
      ptx::mma_commit_elect(&kv_empty[st]);
      ptx::mma_commit_elect(&ds_empty[db]);
    }
    ptx::mma_commit_elect(&acc_full);
  } else {
    const int tid = threadIdx.x, wg = warp >> 2, r = tid & 127;
    const int row = i * kBr + r;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const float tr = valid ? tau[(long long)bh * g.N + row] : kPadTau;
    const float dl = valid ? delta[(long long)bh * g.N + row] : 0.f;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    bool seen = false;   // this warp has seen a non-zero dS (the CTA's first such tile picks K̄, r12)
    // barrier addresses as 32-bit shared offsets, dS buffer index / phase as running counters
    const uint32_t sfull_a = ptx::smem_u32(&s_full), sempty_a = ptx::smem_u32(&s_empty);
    const uint32_t dsf_a0 = ptx::smem_u32(ds_full), dse_a0 = ptx::smem_u32(ds_empty);
    int db = 0;
    uint32_t dph = 0;
    for (int k = 0; k < cnt; ++k) {
      const int jb = list[k];
      const bool masked = (jb + 1) * kBc - 1 > cta_last;
      const int key0 = jb * kBc + wg * CW;
      ptx::mbar_wait_addr(sfull_a, k & 1);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8 * k + 3);
      ptx::tc_fence_after();
      uint32_t pd[WPR];
      const float2 cp2 = make_float2(ap.cp, ap.cp), ntr2 = make_float2(-tr, -tr), ndl2 = make_float2(-dl, -dl);
      // all 64 columns of S and dP at once: the buffers are released right after one TMEM latency, so
      // S/dP(k+1) run on the tensor pipe while this warp computes tile k
      float sa[NH][32], da[NH][32];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        ld32f_nowait(lane_base + t_s + wg * CW + hh * 32, sa[hh]);
        ld32f_nowait(lane_base + t_dp + wg * CW + hh * 32, da[hh]);
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      warp_arrive_addr(sempty_a);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8 * k + 4);
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        const float(&s)[32] = sa[hh];
        const float(&dp)[32] = da[hh];
        auto body = [&](auto masked_c) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float2 x = ffma2(make_float2(s[e], s[e + 1]), cp2, ntr2);
            if constexpr (decltype(masked_c)::value) {
              if (key0 + hh * 32 + e > my_last) x.x = kMaskX;
              if (key0 + hh * 32 + e + 1 > my_last) x.y = kMaskX;
            }
            const float2 g2 = fadd2(make_float2(dp[e], dp[e + 1]), ndl2);
            if constexpr (E == 2 || E == 4) {
              if constexpr (CU) {   // Û (r9)
                uint32_t pb, ub;
                pu_packed<E>(x, pb, ub);
                pd[hh * 16 + (e >> 1)] = mul_bf16x2(ub, ptx::pack_bf16(g2.x, g2.y));
              } else {
                // 2dS = (2u)·(dP − δ), 2u = x + |x| (E = 2) or b + |b|, b = x³ signed: exact doubling, no relu
                const float2 b = E == 2 ? x : fmul2(fmul2(x, fabs2(x)), fabs2(x));
                const float2 ds2 = fmul2(fadd2(b, fabs2(b)), g2);
                pd[hh * 16 + (e >> 1)] = ptx::pack_bf16(ds2.x, ds2.y);
              }
            } else {
              float2 p, u;
              p_and_u2<E>(x, ap, p, u);
              if constexpr (CU)   // Û (r9)
                pd[hh * 16 + (e >> 1)] = mul_bf16x2(ptx::pack_bf16(u.x, u.y), ptx::pack_bf16(g2.x, g2.y));
              else {
                const float2 ds = fmul2(u, g2);
                pd[hh * 16 + (e >> 1)] = ptx::pack_bf16(ds.x, ds.y);
              }
            }
          }
        };
#ifdef ENTMAX_FB_NOMATH
        if (tr == 12345.f)
#endif
        if (masked) body(std::true_type{}); else body(std::false_type{});
      }
      if (!seen) {   // (sign bits masked: U = 0 gives dS = ±0)
        uint32_t orv = 0;
#pragma unroll
        for (int e = 0; e < WPR; ++e) orv |= pd[e];
        seen = __any_sync(0xffffffffu, (orv & 0x7fff7fffu) != 0u);
        if (seen && lane == 0) atomicMin(&s_first, k);
      }
      ptx::mbar_wait_addr(dse_a0 + 8 * db, dph ^ 1u);   // dQ(k−NDS) has consumed this dS buffer
      if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8 * k + 5);
      ptx::tc_fence_after();
      if constexpr (WPR == 32) ptx::tmem_st32(lane_base + t_ds + 64 * db + wg * WPR, pd);
      else ptx::tmem_st16(lane_base + t_ds + 64 * db + wg * WPR, pd);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      warp_arrive_addr(dsf_a0 + 8 * db);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8 * k + 6);
      if (++db == NDS) {
        db = 0;
        dph ^= 1u;
      }
    }
    float rho = 0.f;
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
      uint32_t ra[16];
      ptx::tmem_ld16(lane_base + t_aux, ra);
      ptx::tmem_wait_ld();
      rho = __uint_as_float(ra[0]);
    }
    // leak correction (reading r12): dQ_i = c·Σ_j dŜ_ij (K_j − K̄) = c·(acc_i − ρ_i·K̄), exact in real
    // arithmetic for any K̄ because Σ_j dS_ij = 0 (definition of δ); K̄ = mean key of the
    // CTA's first block with a non-zero dS removes the rounding leak's component along the support's keys
    ptx::named_bar_sync(1, kMath);
    const int kf = s_first;
    constexpr int DS = D / SL;   // dQ columns stored per thread
    const float* kb = (kf == INT_MAX || kbar == nullptr) ? nullptr
                      : kbar + ((long long)bh * g.Tc + list[kf]) * D + wg * DS;
    store_row_bf16_corr<DS>(lane_base + t_dq + wg * DS, dq + g.head_off(bh) + (long long)row * g.sn + wg * DS,
                            ap.scale / kDS, cnt == 0, valid, rho, kb);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ENTMAX_TRACE_K(3, 8003);
  if (warp == MMAW) ptx::tmem_dealloc<512>(tmem);
}

// =====================================================================================
// dK_j, dV_j over 𝒦_j (Alg. 4).  TMEM lanes = the 128 keys of block j.
//   Sᵀ = K_j Q_iᵀ, dPᵀ = V_j dO_iᵀ (SS); Pᵀ and dSᵀ = Uᵀ ⊙ (dPᵀ − δ_i) to TMEM;
//   dV_j += Pᵀ dO_i, dK_j += dSᵀ Q_i (TS); dK scaled by c at the end (Eq. 1).
// MW math warps (8 or 16): warp w owns TMEM lanes 32·(w & 3) and the query-column slice w >> 2 of width
// CW = 128·4/MW; MW = 16 gives four warps per scheduler to hide the per-element latency chains.
// d = 64: Sᵀ [0,128) dPᵀ [128,256) Pᵀ [256,320) dSᵀ [320,384) dV [384,448) dK [448,512), so the
//         next step's Sᵀ/dPᵀ overlap this step's math.
// d = 128: Pᵀ/dSᵀ overwrite each slice's own Sᵀ/dPᵀ columns (dV [256,384), dK [384,512)).
// =====================================================================================
template <int MW>
constexpr int dkdv_threads() { return 32 * MW + 64; }

template <int D, int E, bool CU, int MW>
__global__ void __launch_bounds__(dkdv_threads<MW>(), 1)
dkdv_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
            const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo, Geom g, AlphaParams ap,
            const float* __restrict__ td, const int32_t* __restrict__ col_cnt,
            const int32_t* __restrict__ col_idx, float* __restrict__ kbar, __nv_bfloat16* __restrict__ dk,
            __nv_bfloat16* __restrict__ dv) {
  using C = Cfg<D>;
  constexpr bool ALIAS = (D == 128);
  constexpr int NST = (D == 64) ? 5 : 2;   // Q/dO/τ/δ stages
  constexpr uint32_t STAGE = 2 * C::TILE + 1024;   // Q_i | dO_i | τ_i[128] | δ_i[128]
  constexpr float kDS = ((E == 2 || E == 4) && !CU) ? 2.f : 1.f;   // the stored dSᵀ is kDS·dSᵀ (exact doubling)
  constexpr int kMath = 32 * MW;
  constexpr int SL = MW / 4;           // query-column slices
  constexpr int CW = 128 / SL;         // query columns per thread
  constexpr int NH = CW / 32;          // 32-column halves per thread
  constexpr int WPR = CW / 2;          // bf16x2 words per thread of Pᵀ / dSᵀ
  constexpr int KPS = CW / 16;         // MMA k-steps per slice
  constexpr int PROD = MW, MMAW = MW + 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* sStage = sV + C::TILE;
  __shared__ __align__(8) uint64_t bar_kv, qd_full[NST], qd_empty[NST], s_full, s_empty, p_full, p_empty, acc_full;
  __shared__ uint32_t tmem_base_sh;

  const int j = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lj = (long long)bh * g.Tc + j;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_kv, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&qd_full[s], 1);
      ptx::mbar_init(&qd_empty[s], 1);
    }
    ptx::mbar_init(&s_full, 1);
    ptx::mbar_init(&s_empty, MW);
    ptx::mbar_init(&p_full, MW);
    ptx::mbar_init(&p_empty, 1);
    ptx::mbar_init(&acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8002);
  if (warp == MMAW) ptx::tmem_alloc<512>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t t_s = tmem, t_dp = tmem + 128;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // δ and the 𝒦 tables are complete
  const bool dense = col_idx == nullptr;   // unmasked mode: every query block that sees key block j
  const int i0 = g.causal ? (j * kBc) / kBr : 0;
  const int cnt = dense ? g.Tr - i0 : col_cnt[lj];
  const BlockList list{dense ? nullptr : col_idx + lj * g.Tr, i0};
  const uint32_t t_dv = tmem + (ALIAS ? 256 : 384), t_dk = t_dv + D;
  // k-step ks (16 query columns = 8 TMEM words) of Pᵀ / dSᵀ: slice ks / KPS, word 8·(ks % KPS) of it
  auto pt_col = [&](int ks) {
    return ALIAS ? t_s + CW * (ks / KPS) + 8 * (ks % KPS) : tmem + 256 + 8 * ks;
  };
  auto dst_col = [&](int ks) {
    return ALIAS ? t_dp + CW * (ks / KPS) + 8 * (ks % KPS) : tmem + 320 + 8 * ks;
  };

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
      ENTMAX_TRACE_K(2, 8 * k + 7);
      // τ_i and δ_i of the block's 128 rows (+∞ / 0 past N) with one bulk copy from the staging array the
      // δ kernel wrote — asynchronous like the tiles, so the producer never waits on a global load
      ENTMAX_TRACE_K(2, 4224 + k);
      ptx::mbar_arrive_expect_tx_elect(&qd_full[st], 2 * C::TILE + 2 * kBr * 4);
      ptx::bulk_load_elect(stg + 2 * C::TILE, td + ((long long)bh * g.Tr + ib) * (2 * kBr), 2 * kBr * 4, &qd_full[st]);
      tma_tile<D>(stg, &tq, &qd_full[st], ib * kBr, h, b);
      tma_tile<D>(stg + C::TILE, &tdo, &qd_full[st], ib * kBr, h, b);
    }
  } else if (warp == MMAW) {
    ptx::mbar_wait(&bar_kv, 0);
    auto issue_sdp = [&](int k) {
      const int st = k % NST;
      const uint8_t* stg = sStage + st * STAGE;
      ptx::mbar_wait(&qd_full[st], (k / NST) & 1);
      ENTMAX_TRACE_K(2, 4096 + k);
      if (!ALIAS) ptx::mbar_wait(&s_empty, (k & 1) ^ 1);
      ENTMAX_TRACE_K(2, 4160 + k);
      ptx::tc_fence_after();
      mma_rows_x_rows<D>(t_s, sK, stg, false);             // Sᵀ  = K_j Q_iᵀ
      mma_rows_x_rows<D>(t_dp, sV, stg + C::TILE, false);  // dPᵀ = V_j dO_iᵀ
      ptx::mma_commit_elect(&s_full);
      ENTMAX_TRACE_K(2, 8 * k + 0);
    };
    if (cnt > 0) issue_sdp(0);
    for (int k = 0; k < cnt; ++k) {
      if (!ALIAS && k + 1 < cnt) issue_sdp(k + 1);
      const int st = k % NST;
      const uint8_t* stg = sStage + st * STAGE;
      ptx::mbar_wait(&p_full, k & 1);
      ENTMAX_TRACE_K(2, 8 * k + 1);
      ptx::tc_fence_after();
      mma_tmem_x_tile<D>(t_dv, pt_col, stg + C::TILE, k > 0);   // dV += Pᵀ dO_i
      mma_tmem_x_tile<D>(t_dk, dst_col, stg, k > 0);            // dK += dSᵀ Q_i
      ptx::mma_commit_elect(&qd_empty[st]);
      if (!ALIAS) ptx::mma_commit_elect(&p_empty);   // (aliased Pᵀ/dSᵀ: the next Sᵀ MMA orders it)
      if (ALIAS && k + 1 < cnt) issue_sdp(k + 1);
    }
    ptx::mma_commit_elect(&acc_full);
    ENTMAX_TRACE_K(2, 8001);
  } else {
    const int tid = threadIdx.x, wg = warp >> 2, r = tid & 127;
    const int key = j * kBc + r;
    const bool valid = key < g.N;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    // per-tile addressing kept out of the loop body: shared addresses as 32-bit offsets, the stage index
    // and phase as running counters; the 𝒦 list is read only for the causal diagonal test (the list is
    // ascending from i0 = j, so only its first entry can be the diagonal block)
    const uint32_t stage_a0 = ptx::smem_u32(sStage) + 2 * C::TILE + wg * (CW * 4);
    const uint32_t qdf_a0 = ptx::smem_u32(qd_full), sfull_a = ptx::smem_u32(&s_full);
    const bool diag0 = g.causal && cnt > 0 && list[0] == j;
    int st = 0;
    uint32_t qph = 0;
    for (int k = 0; k < cnt; ++k) {
      const uint32_t tq4 = stage_a0 + st * STAGE;   // τ_i (float4 units below)
      const uint32_t dl4 = tq4 + 512;               // δ_i
      const bool diag = diag0 && k == 0;            // queries below the key inside the diagonal block
      ptx::mbar_wait_addr(qdf_a0 + 8 * st, qph);    // τ_i, δ_i staged by the producer warp
      if (++st == NST) {
        st = 0;
        qph ^= 1u;
      }
      ptx::mbar_wait_addr(sfull_a, k & 1);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8 * k + 3);
      ptx::tc_fence_after();
      uint32_t pp[WPR], pd[WPR];
      // all of this thread's columns of Sᵀ and dPᵀ are read at once, so the MMA warp can start
      // Sᵀ/dPᵀ(k+1) while this warp still computes tile k
      float sa[NH][32], da[NH][32];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        ld32f_nowait(lane_base + t_s + wg * CW + hh * 32, sa[hh]);
        ld32f_nowait(lane_base + t_dp + wg * CW + hh * 32, da[hh]);
      }
      ptx::tmem_wait_ld();
      if (!ALIAS) {
        ptx::tc_fence_before();
        warp_arrive(&s_empty);
      }
      if (lane == 0) ENTMAX_TRACE_K(2, 4288 + 8 * k + (warp & 7));
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        const float(&s)[32] = sa[hh];
        const float(&dp)[32] = da[hh];
        auto body = [&](auto masked_c) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 t4 = ld_shared_f4(tq4 + (hh * 8 + q4) * 16), d4 = ld_shared_f4(dl4 + (hh * 8 + q4) * 16);
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const float2 tq2 = e == 0 ? make_float2(-t4.x, -t4.y) : make_float2(-t4.z, -t4.w);
              const float2 dq2 = e == 0 ? make_float2(-d4.x, -d4.y) : make_float2(-d4.z, -d4.w);
              float2 x = ffma2(make_float2(s[q4 * 4 + e], s[q4 * 4 + e + 1]), make_float2(ap.cp, ap.cp), tq2);
              if constexpr (decltype(masked_c)::value) {
                const int ql = wg * CW + hh * 32 + q4 * 4 + e;
                if (!valid || (diag && ql < r)) x.x = kMaskX;
                if (!valid || (diag && ql + 1 < r)) x.y = kMaskX;
              }
              const float2 g2 = fadd2(make_float2(dp[q4 * 4 + e], dp[q4 * 4 + e + 1]), dq2);
              const int w = hh * 16 + q4 * 2 + (e >> 1);
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
#ifdef ENTMAX_FB_NOMATH
        if (key == -12345)
#endif
        if (!valid || diag) body(std::true_type{}); else body(std::false_type{});
      }
      if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8 * k + 4);
      if (!ALIAS) {
        ptx::mbar_wait(&p_empty, (k & 1) ^ 1);   // dV/dK(k−1) have consumed the previous Pᵀ, dSᵀ
        ptx::tc_fence_after();
      }
      if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8 * k + 5);
      if constexpr (WPR == 32) {
        ptx::tmem_st32(lane_base + pt_col(wg * KPS), pp);
        ptx::tmem_st32(lane_base + dst_col(wg * KPS), pd);
      } else {
        ptx::tmem_st16(lane_base + pt_col(wg * KPS), pp);
        ptx::tmem_st16(lane_base + dst_col(wg * KPS), pd);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      warp_arrive(&p_full);
      if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8 * k + 6);
    }
    if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8000);
    if (cnt > 0) {
      ptx::mbar_wait(&acc_full, 0);
      ptx::tc_fence_after();
    }
    constexpr int DS = D / SL;   // dK / dV columns stored per thread
    const long long off = g.head_off(bh) + (long long)(valid ? key : 0) * g.sn + wg * DS;
    store_cols_bf16<DS>(lane_base + t_dv + wg * DS, dv + off, 1.0f, cnt == 0, valid);
    store_cols_bf16<DS>(lane_base + t_dk + wg * DS, dk + off, ap.scale / kDS, cnt == 0, valid);
    if (kbar != nullptr) {
      // K̄_j = mean of the block's keys (fp32) for the dQ kernel's leak correction (reading r12), from the
      // K tile this CTA holds in shared memory (rows past N are TMA zero fill).  Thread → (16-byte unit u of
      // a row, row phase rp); partial sums reduced through the (now idle) stage buffers.
      constexpr int UNITS = D / 8, RP = kMath / UNITS;
      ptx::mbar_wait(&bar_kv, 0);
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
      float* red = reinterpret_cast<float*>(sStage);   // [RP][D]
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
  if (threadIdx.x == 0) ENTMAX_TRACE_K(2, 8003);
  if (warp == MMAW) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace sm100
}  // namespace entmax
