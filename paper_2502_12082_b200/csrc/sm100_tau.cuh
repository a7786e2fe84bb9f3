// sm100_tau.cuh — τ by Halley-bisection with on-chip candidate compaction (sm_100a).
//
// Paper: Alg. 1 per row, Alg. 3 per query block: one pass for the row
// max, then T passes accumulating f, f', f'' (Eqs. 3, 6, 7) over all K blocks (Eq. 8).
//
// B200 design (same result, fewer passes): after pass 0 (row max m, bracket τ_lo = m − 1), pass 1
// streams the K blocks once more and copies every score with (α−1)c·s > τ_lo into a per-row list
// in shared memory.  Every other element has x = z − τ <= z − τ_lo <= 0 for every iterate τ >= τ_lo
// (the bracket only moves up), so it contributes exact zeros to f, f', f'' (reading c7) — the T
// Halley-bisection iterations then run on the compact lists without recomputing S.  The same
// lists, tested against the final τ with the kernels' own fma(s, c', −τ) > 0, give the exact
// block mask, so the output kernel only visits active blocks.  If a row's list overflows (wide
// supports, small α), the CTA falls back to streaming passes 2..T+1 over the candidate blocks
// (blocks holding any element above τ_lo), i.e. Alg. 3 restricted to those blocks.
//
// Warp roles (320 threads): warps 0-7 math (thread t: row t & 127, column half t >> 7 of each
// 128-key tile; warp w reads TMEM lanes 32·(w & 3)), warp 8 TMA producer, warp 9 MMA issuer.
#pragma once

#include "sm100_kernels.cuh"
#include "trace.cuh"

namespace entmax {
namespace sm100 {

constexpr int kTauThreads = 320;
constexpr int kTauMath = 256;
constexpr int kTauCap = 80;  // list slots per (row, column half); the count has a heavy tail
constexpr int kTauSBuf = 4;  // S tiles in flight in TMEM (4 × 128 columns)

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <int D>
struct TauSmem {
  static constexpr int NST = (D == 64) ? 4 : 2;   // K-tile ring depth
  static constexpr size_t tiles = (size_t)(1 + NST) * Cfg<D>::TILE;
  static constexpr size_t lists = (size_t)(kTauCap + 1) * kTauMath * (4 + 2);   // + scratch slot
  static constexpr size_t fixed = 1024 + tiles + lists + kTauMath * 4 * 4;  // + exchange scratch
  static size_t bytes(int Tc) { return fixed + 4 * (size_t)Tc + 64; }   // cflag, aflag (u8) + cblk (u16)
};

// Launched as clusters of two CTAs = two adjacent query blocks of the same head, which stream the
// same K blocks: each CTA TMA-loads half of every K tile (64 rows) with .multicast::cluster, so an SM
// issues 8 KB per tile instead of 16 KB (TMA issue on the SM is what slows the tensor pipe down,
// see DESIGN.md §6).  MMA completions are committed to the empty barriers of both CTAs.
// `tk` is a tensor map with 64-row boxes.  Grid x is rounded up to even; a CTA past T_r streams and
// computes but writes nothing.
template <int D, int E>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTauThreads, 1)
tau_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk, Geom g, AlphaParams ap,
           int n_iter, float* __restrict__ tau_out, int32_t* __restrict__ cand_cnt, int32_t* __restrict__ cand_idx) {
  using C = Cfg<D>;
  using SM = TauSmem<D>;
  constexpr int NST = SM::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::TILE;
  float* list_s = reinterpret_cast<float*>(sK + NST * C::TILE);           // [CAP+1][256]
  uint16_t* list_j = reinterpret_cast<uint16_t*>(list_s + (kTauCap + 1) * kTauMath);  // [CAP+1][256]
  float* xch = reinterpret_cast<float*>(list_j + (kTauCap + 1) * kTauMath);      // [4][256] exchange
  uint8_t* cflag = reinterpret_cast<uint8_t*>(xch + 4 * kTauMath);         // [Tc] candidate blocks (τ_lo)
  uint8_t* aflag = cflag + g.Tc;                                           // [Tc] exact active blocks
  uint16_t* cblk = reinterpret_cast<uint16_t*>(aflag + g.Tc);            // [Tc] fallback block list (2·Tc even)
  __shared__ __align__(8) uint64_t bar_q, k_full[NST], k_empty[NST], s_full[kTauSBuf], s_empty[kTauSBuf], dec_bar,
      x_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_fallback, s_ncb, s_overflow, s_peer_overflow;

  const int i = blockIdx.x, bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank(), peer = rank ^ 1u;
  const bool real_cta = i < g.Tr;
  const int nkb = g.visible_kblocks(min((i | 1), g.Tr - 1));   // identical for both CTAs of the pair
  const long long li = (long long)bh * g.Tr + i;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 2);      // one MMA commit from each CTA of the pair
    }
    for (int s = 0; s < kTauSBuf; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], 8);
    }
    ptx::mbar_init(&dec_bar, 1);
    ptx::mbar_init(&x_bar, 1);
    ptx::fence_mbar_init();
    s_overflow = 0;
  }
  for (int j = threadIdx.x; j < g.Tc; j += blockDim.x) {
    cflag[j] = 0;
    aflag[j] = 0;
  }
  if (warp == 9) ptx::tmem_alloc<128 * kTauSBuf>(&tmem_base_sh);
  ptx::tc_fence_before();
  ptx::cluster_sync();   // both CTAs' barriers exist before any multicast targets them
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 8) {
    // ---------------------------------------------------------------- TMA producer
    ptx::tma_prefetch_desc(&tq);
    ptx::tma_prefetch_desc(&tk);
    ptx::mbar_arrive_expect_tx_elect(&bar_q, C::TILE);
    tma_tile<D>(sQ, &tq, &bar_q, i * kBr, h, b);
    int k = 0;
    auto load = [&](int j) {
      const int st = k % NST;
      ptx::mbar_wait(&k_empty[st], ((k / NST) & 1) ^ 1);
      ENTMAX_TRACE_EV(6144 + k);
      ptx::mbar_arrive_expect_tx_elect(&k_full[st], C::TILE);   // both halves land here
#pragma unroll
      for (int c = 0; c < C::KCH; ++c)
        ptx::tma_load_4d_mc_elect(sK + st * C::TILE + c * kChunkBytes + rank * (kChunkBytes / 2), &tk, &k_full[st], c * 64,
                            j * kBc + (int)rank * 64, h, b, 0x3);
      ++k;
    };
    for (int p = 0; p < 2; ++p)
      for (int j = 0; j < nkb; ++j) load(j);
    ptx::mbar_wait(&dec_bar, 0);
    if (s_fallback)
      for (int t = 0; t < n_iter; ++t)
        for (int c = 0; c < s_ncb; ++c) load(cblk[c]);
  } else if (warp == 9) {
    // ---------------------------------------------------------------- MMA issuer
    ptx::mbar_wait(&bar_q, 0);
    int k = 0;
    auto mma = [&]() {
      const int st = k % NST, sb = k % kTauSBuf;
      ENTMAX_TRACE_EV(4 * k);
      ptx::mbar_wait(&k_full[st], (k / NST) & 1);
      ENTMAX_TRACE_EV(4 * k + 1);
      ptx::mbar_wait(&s_empty[sb], ((k / kTauSBuf) & 1) ^ 1);
      ENTMAX_TRACE_EV(4 * k + 2);
      ptx::tc_fence_after();
      mma_rows_x_rows<D>(tmem + sb * 128, sQ, sK + st * C::TILE, false);
      ptx::mma_commit_mc_elect(&k_empty[st], 0x3);
      ptx::mma_commit_elect(&s_full[sb]);
      ++k;
    };
    for (int p = 0; p < 2 * nkb; ++p) mma();
    ptx::mbar_wait(&dec_bar, 0);
    if (s_fallback)
      for (int p = 0; p < n_iter * s_ncb; ++p) mma();
  } else {
    // ---------------------------------------------------------------- math warps (256 threads)
    const int tid = threadIdx.x;
    const int r = tid & 127, hf = tid >> 7;
    const int row = i * kBr + r;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + hf * 64;
    int k = 0;

    // read this thread's 64 scores of step k (columns hf*64 .. +63 of key block j), masked
    auto read_tile = [&](int j, float (&s)[64]) {
      const int sb = k % kTauSBuf;
      if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * k);
      ptx::mbar_wait(&s_full[sb], (k / kTauSBuf) & 1);
      if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * k + 1);
      ptx::tc_fence_after();
      uint32_t ra[32], rb[32];
#ifdef ENTMAX_TRACE_NOLD
#pragma unroll
      for (int e = 0; e < 32; ++e) ra[e] = rb[e] = 0u;
#else
      ptx::tmem_ld32(lane_base + sb * 128, ra);
      ptx::tmem_ld32(lane_base + sb * 128 + 32, rb);
      ptx::tmem_wait_ld();
#endif
      ptx::tc_fence_before();
      warp_arrive(&s_empty[sb]);
      if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * k + 2);
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        s[e] = __uint_as_float(ra[e]);
        s[32 + e] = __uint_as_float(rb[e]);
      }
      if ((j + 1) * kBc - 1 > cta_last) {
        const int key0 = j * kBc + hf * 64;
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (key0 + e > my_last) s[e] = -INFINITY;
      }
      ++k;
    };

    // ---- pass 0: row max (Alg. 1 line 4)
    float smax = -INFINITY;
    for (int j = 0; j < nkb; ++j) {
      float s[64];
      read_tile(j, s);
#pragma unroll
      for (int e = 0; e < 64; e += 2) smax = fmax3(smax, s[e], s[e + 1]);
    }
    xch[tid] = smax;
    ptx::named_bar_sync(1, kTauMath);
    smax = fmaxf(xch[r], xch[128 + r]);
    const float n_vis = g.causal ? (float)(row + 1) : (float)g.N;
    RowState rs = bracket_init(smax * ap.cp, n_vis, ap.alpha);
    // conservative score threshold: s <= thr ⇒ fma(s, c', −τ_lo) <= 0 (margin >> fma rounding)
    const float thr = (rs.lo - fmaxf(fabsf(rs.lo), 1e-6f) * 3.0e-6f) / ap.cp;

    // ---- pass 1: compact the candidates z > τ_lo into this thread's list
    int cnt = 0;
    for (int j = 0; j < nkb; ++j) {
      float s[64];
      read_tile(j, s);
      // groups of 8 keys: a group max (FMNMX3) decides whether the short, branch-free append
      // runs; candidates are rare (~1e-3 of the keys for Gaussian rows at α = 1.5)
      const float thr_v = valid ? thr : INFINITY;
      bool any = false;
#pragma unroll
      for (int gq = 0; gq < 8; ++gq) {
        const float* sg = s + 8 * gq;
        const float gm = fmax3(fmax3(sg[0], sg[1], sg[2]), fmax3(sg[3], sg[4], sg[5]), fmaxf(sg[6], sg[7]));
        if (gm > thr_v) {
          any = true;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const bool p = sg[e] > thr_v;
            const int slot = min(cnt, kTauCap);            // slot kTauCap is a scratch slot
            if (p) {
              list_s[slot * kTauMath + tid] = sg[e];
              list_j[slot * kTauMath + tid] = (uint16_t)j;
            }
            cnt += p ? 1 : 0;
          }
        }
      }
      if (__any_sync(0xffffffffu, any) && lane == 0) cflag[j] = 1;
    }
    if (cnt > kTauCap) s_overflow = 1;
    ptx::named_bar_sync(1, kTauMath);
    // the pair shares the K stream, so the fallback decision is exchanged and made jointly
    if (tid == 0) {
      ptx::st_cluster_u32(ptx::mapa(ptx::smem_u32(&s_peer_overflow), peer), (uint32_t)s_overflow);
      ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&x_bar), peer));
      ptx::mbar_wait_cluster(&x_bar, 0);
      s_fallback = (s_overflow | s_peer_overflow) ? 1 : 0;
    }
    ptx::named_bar_sync(1, kTauMath);
    const bool fallback = s_fallback != 0;

    if (!fallback) {
      // ---- T iterations of Alg. 1 on the compact lists (one thread per row: hf == 0)
      xch[tid] = __int_as_float(cnt);
      ptx::named_bar_sync(1, kTauMath);
      if (hf == 0) {
        const int c0 = cnt, c1 = __float_as_int(xch[128 + r]);
        for (int t = 0; t < n_iter; ++t) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f;
          for (int c = 0; c < c0; ++c) accum_f<E>(fmaf(list_s[c * kTauMath + r], ap.cp, -rs.tau), ap, a0, a1, a2);
          for (int c = 0; c < c1; ++c)
            accum_f<E>(fmaf(list_s[c * kTauMath + 128 + r], ap.cp, -rs.tau), ap, a0, a1, a2);
          alg1_update(rs, a0, a1, a2, ap);
        }
        if (valid) {
          tau_out[(long long)bh * g.N + row] = rs.tau;
          // exact block activity from the final τ (same fma test as the output kernel)
          for (int c = 0; c < c0; ++c)
            if (fmaf(list_s[c * kTauMath + r], ap.cp, -rs.tau) > 0.f) aflag[list_j[c * kTauMath + r]] = 1;
          for (int c = 0; c < c1; ++c)
            if (fmaf(list_s[c * kTauMath + 128 + r], ap.cp, -rs.tau) > 0.f)
              aflag[list_j[c * kTauMath + 128 + r]] = 1;
        }
      }
      ptx::named_bar_sync(1, kTauMath);
      if (warp == 0 && real_cta) {
        const int n = compact_flags(aflag, nkb, cand_idx + li * g.Tc);
        if (lane == 0) cand_cnt[li] = n;
      }
      if (tid == 0) {
        __threadfence_block();
        ptx::mbar_arrive(&dec_bar);
      }
    } else {
      // ---- fallback: streaming Alg. 3 passes over every visible block (the pair streams the same
      // blocks, so no per-CTA pruning); the output kernel gets this CTA's τ_lo candidate blocks
      if (warp == 0) {
        for (int c = lane; c < nkb; c += 32) cblk[c] = (uint16_t)c;
        if (real_cta) {
          const int n = compact_flags(cflag, nkb, cand_idx + li * g.Tc);
          if (lane == 0) cand_cnt[li] = n;
        }
        __syncwarp();
        if (lane == 0) {
          s_ncb = nkb;
          __threadfence_block();
          ptx::mbar_arrive(&dec_bar);
        }
      }
      ptx::named_bar_sync(1, kTauMath);
      const int ncb = s_ncb;
      for (int t = 0; t < n_iter; ++t) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
        for (int c = 0; c < ncb; ++c) {
          float s[64];
          read_tile(cblk[c], s);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            float cm = s[32 * q];
#pragma unroll
            for (int e = 1; e < 32; e += 2) cm = fmax3(cm, s[32 * q + e], s[32 * q + e + 1]);
            if (__any_sync(0xffffffffu, fmaf(cm, ap.cp, -rs.tau) > 0.f)) {
#pragma unroll
              for (int e = 0; e < 32; ++e) accum_f<E>(fmaf(s[32 * q + e], ap.cp, -rs.tau), ap, a0, a1, a2);
            }
          }
        }
        // combine the two column halves in a fixed order (identical update in both threads)
        ptx::named_bar_sync(1, kTauMath);
        xch[tid] = a0;
        xch[kTauMath + tid] = a1;
        xch[2 * kTauMath + tid] = a2;
        ptx::named_bar_sync(1, kTauMath);
        a0 = xch[r] + xch[128 + r];
        a1 = xch[kTauMath + r] + xch[kTauMath + 128 + r];
        a2 = xch[2 * kTauMath + r] + xch[2 * kTauMath + 128 + r];
        alg1_update(rs, a0, a1, a2, ap);
      }
      if (hf == 0 && valid) tau_out[(long long)bh * g.N + row] = rs.tau;
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();   // no CTA leaves while its peer may still multicast into it
  if (warp == 9) ptx::tmem_dealloc<128 * kTauSBuf>(tmem);
}

}  // namespace sm100
}  // namespace entmax
