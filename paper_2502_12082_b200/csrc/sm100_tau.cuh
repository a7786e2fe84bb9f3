// sm100_tau.cuh — τ by Halley-bisection with on-chip candidate compaction (sm_100a).
//
// Paper: Alg. 1 per row, Alg. 3 per query block: one pass for the row
// max, then T passes accumulating f, f', f'' (Eqs. 3, 6, 7) over all K blocks (Eq. 8).
//
// B200 design (same result, one pass over K in the common case): the K blocks stream once; the
// threads of a row keep a running max m_run of the row and append every score with
// c'·s > τ_lo(m_run) = c'·m_run − 1 to the row's candidate list in shared memory.  m_run <= m, so
// τ_lo(m_run) <= τ_lo(m) and every score the final filter needs is kept; everything else has
// x = z − τ <= z − τ_lo(m) <= 0 for every iterate τ >= τ_lo(m) (the bracket only moves up) and
// contributes exact zeros to f, f', f'' (reading c7).  The T Halley-bisection iterations then run
// on the lists without recomputing S.  The same lists, tested against the final τ with the kernels'
// own fma(s, c', −τ) > 0, give the exact block mask, so the output kernel only visits active blocks.
// The first W blocks only raise the running max and are streamed again at the end (fewer transient
// candidates).  Each row list is split into four private quarters, one per thread of the row, so an
// append is a plain shared store at a register counter (no atomics) and every thread's list keeps
// the stream order; the iteration sums are fixed-point (FxSum below), so τ is bitwise reproducible
// (entries appended under a racy, lower running threshold are <= τ_lo(m) and add nothing).  Overflow (a row list is finite): tier 1 streams K once more with the exact threshold
// τ_lo(m); tier 2, if even that overflows (wide supports, small α), streams T more passes over all
// visible blocks — Alg. 3 itself.
// Warp roles (576 threads): warps 0-15 math in four groups of four (thread t: row t & 127; group
// t >> 7 owns S buffer t >> 7 and processes every fourth tile of the stream, all 128 columns of it in
// four 32-column TMEM loads; warp w reads TMEM lanes 32·(w & 3)), so four tiles are in processing at
// once and a warp's per-tile overheads cover a whole row segment; warp 16 TMA producer, warp 17 MMA
// issuer.
#pragma once

#include "sm100_kernels.cuh"
#include "trace.cuh"

namespace entmax {
namespace sm100 {

constexpr int kTauMathWarps = 16;
constexpr int kTauMath = 32 * kTauMathWarps;
constexpr int kTauThreads = kTauMath + 64;
constexpr int kTauSBuf = 4;  // S tiles in flight in TMEM (4 × 128 columns)

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// Private-list append: if v > thr, store v at [as] and the u16 tag at [aj] (only while as < end) and
// advance both by one slot.  Lists are slot-major ([slot][128 rows]: 512 B per value slot, 256 B per
// tag slot) so the lanes (rows) of a warp store to consecutive words; as keeps advancing past `end`
// so the list length (and an overflow) is (as − start) / 512.
__device__ __forceinline__ void list_append(uint32_t& as, uint32_t& aj, uint32_t end, float v, float thr,
                                            uint32_t tag) {
  asm volatile(
      "{.reg .pred q, w;\n\tsetp.gt.f32 q, %2, %3;\n\tsetp.lt.and.u32 w, %0, %5, q;\n\t"
      "@w st.shared.f32 [%0], %2;\n\t@w st.shared.u16 [%1], %4;\n\t"
      "@q add.u32 %0, %0, 512;\n\t@q add.u32 %1, %1, 256;\n\t}"
      : "+r"(as), "+r"(aj)
      : "f"(v), "f"(thr), "h"((unsigned short)tag), "r"(end)
      : "memory");
}

// Order-independent sums of Eqs. 3/6/7: every term is rounded once to fixed point and the integers
// add exactly, so τ is bitwise the same whatever partition and order the contributing scores were
// visited in — the online lists, the exact-threshold rebuild (tier 1) and the streaming passes (tier 2)
// all give identical bits, and the (racy, timing-dependent) choice between them cannot change the
// result.  E ∈ {1, 2, 4}: every term lies in [0, 1] (x <= m·c′ − τ_lo = 1), and its 2^-23 fixed-point
// value is the mantissa of t + 1 (one FADD, exact RN rounding) — unit 2^-23.  Generic α: unit 2^-32 for
// [x]_+^e, [x]_+^{e−1} ∈ [0, 1]; [x]_+^{e−2} exceeds 1 when e < 2 (α > 1.5): unit 2^-20, clamped at 2^30.
struct FxSum {
  unsigned long long q0, q1, q2;
};
__device__ __forceinline__ uint32_t fx23(float t) { return __float_as_uint(t + 1.0f) - 0x3f800000u; }
// terms of one x into 32-bit partials (E != 0; x <= 0 gives zero terms and fx23(0) = 0 exactly;
// <= 256 terms per partial)
template <int E>
__device__ __forceinline__ void accum_fx32(float x, const AlphaParams& ap, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  float t0 = 0.f, t1 = 0.f, t2 = 0.f;
  accum_f<E>(x, ap, t0, t1, t2);
  p0 += fx23(t0);
  p1 += fx23(t1);
  p2 += fx23(t2);
}
// accum_fx32<E> on a pair of x in packed f32x2 (E = 1, 2, 4), RAW: every term adds bits(t + 1) — the caller
// subtracts 0x3f800000 per term (mod 2³²) once at the end.  r = x + |x| = 2x₊ exactly, and the powers of r
// are scaled back by exact powers of two inside the fma that forms t + 1, so the terms are bitwise those
// of accum_fx32 (where a power-of-two scaling would round differently — subnormal x₊² — every term is 0
// anyway); [x > 0] = min(r · 2¹⁰⁰, 1) (r ≥ 2⁻⁵⁰ whenever x > 0).  x must be finite (pads: −1e30).
template <int E>
__device__ __forceinline__ void accum_fx32_pair_raw(float2 x, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  const float2 one2 = make_float2(1.0f, 1.0f);
  const float2 r = fadd2(x, fabs2(x));
  auto bits2 = [](float2 v) { return __float_as_uint(v.x) + __float_as_uint(v.y); };
  auto ind1 = [&]() {   // [x > 0] + 1
    const float2 g = fmul2(r, make_float2(0x1p100f, 0x1p100f));
    return fadd2(make_float2(fminf(g.x, 1.0f), fminf(g.y, 1.0f)), one2);
  };
  if constexpr (E == 4) {
    const float2 r2 = fmul2(r, r);
    p0 += bits2(ffma2(fmul2(r2, r2), make_float2(0.0625f, 0.0625f), one2));
    p1 += bits2(ffma2(fmul2(r2, r), make_float2(0.125f, 0.125f), one2));
    p2 += bits2(ffma2(r2, make_float2(0.25f, 0.25f), one2));
  } else if constexpr (E == 2) {
    p0 += bits2(ffma2(fmul2(r, r), make_float2(0.25f, 0.25f), one2));
    p1 += bits2(ffma2(r, make_float2(0.5f, 0.5f), one2));
    p2 += bits2(ind1());
  } else {   // E == 1: x₊, [x > 0], 0
    p0 += bits2(ffma2(r, make_float2(0.5f, 0.5f), one2));
    p1 += bits2(ind1());
    p2 += 2u * 0x3f800000u;   // t = 0 (kept in the raw convention)
  }
}

template <int E>
__device__ __forceinline__ void accum_fx(float x, const AlphaParams& ap, float u2, FxSum& q) {
  if constexpr (E != 0) {
    uint32_t p0 = 0, p1 = 0, p2 = 0;
    accum_fx32<E>(x, ap, p0, p1, p2);
    q.q0 += p0;
    q.q1 += p1;
    q.q2 += p2;
  } else {
    float t0 = 0.f, t1 = 0.f, t2 = 0.f;
    accum_f<E>(x, ap, t0, t1, t2);
    q.q0 += __float2ull_rn(t0 * 4294967296.0f);
    q.q1 += __float2ull_rn(t1 * 4294967296.0f);
    q.q2 += __float2ull_rn(fminf(t2, 1073741824.0f) * u2);
  }
}

template <int D>
struct TauSmem {
#ifdef ENTMAX_TAU_NST   // diagnostics override
  static constexpr int NST = (D == 64) ? ENTMAX_TAU_NST : 2;
#else
  static constexpr int NST = (D == 64) ? 3 : 2;   // K-tile ring depth
#endif
  // list slots per row: the online pass appends ~37 scores per row on average for the paper's
  // Gaussian rows at N = 8192 (max ~140); the exact-threshold count has a heavy tail (DESIGN.md §τ)
#ifdef ENTMAX_TAU_CAP
  static constexpr int CAP = (D == 64) ? ENTMAX_TAU_CAP : 144;
#else
  static constexpr int CAP = (D == 64) ? 188 : 144;
#endif
  static constexpr int CAPQ = CAP / 4;                                // private slots per thread
  static constexpr size_t tiles = (size_t)(1 + NST) * Cfg<D>::TILE;
  static constexpr size_t lists = (size_t)CAP * kBr * (4 + 2);     // score f32, key block u16
  static constexpr size_t fixed = 1024 + tiles + lists + 3 * kTauMath * 8 + 2 * kBr * 4;
  static size_t bytes(int Tc) { return fixed + 2 * (size_t)Tc + 64; }   // cflag, aflag (u8)
};

// One CTA per 128-row query block, no cluster: the K tiles stream by plain TMA into a private ring (a
// 2-CTA cluster sharing every K tile by multicast measured 4-11 % slower: the pair's stage reuse waits
// for the slower CTA).  `tk` is a tensor map with 128-row boxes.
template <int D, int E>
__global__ void __launch_bounds__(kTauThreads, 1)
tau_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk, Geom g, AlphaParams ap,
           int n_iter, float* __restrict__ tau_out, int32_t* __restrict__ cand_cnt, int32_t* __restrict__ cand_idx) {
  using C = Cfg<D>;
  using SM = TauSmem<D>;
  constexpr int NST = SM::NST;
  constexpr int kCap = SM::CAP;
  constexpr int kCapQ = SM::CAPQ;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::TILE;
  float* list_s = reinterpret_cast<float*>(sK + NST * C::TILE);            // [CAP][128] scores
  uint16_t* list_j = reinterpret_cast<uint16_t*>(list_s + kCap * kBr);      // [CAP][128] key block
  float* xch = reinterpret_cast<float*>(list_j + kCap * kBr);               // [3][512] exchange (8-byte slots)
  float* mshare = xch + 6 * kTauMath;                                        // [128] running row maxima
  int* rowcnt = reinterpret_cast<int*>(mshare + kBr);                        // [128] (spare)
  uint8_t* cflag = reinterpret_cast<uint8_t*>(rowcnt + kBr);                 // [Tc] candidate blocks (τ_lo)
  uint8_t* aflag = cflag + g.Tc;                                             // [Tc] exact active blocks
  __shared__ __align__(8) uint64_t bar_q, k_full[NST], k_empty[NST], s_full[kTauSBuf], s_empty[kTauSBuf], dec_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_fallback, s_overflow;

  // causal: the longest query blocks first (the block scheduler issues low indices first)
  const int i = g.causal ? g.Tr - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int bh = blockIdx.y;
  const int b = bh / g.H, h = bh - b * g.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = g.visible_kblocks(i);
  const bool real_cta = i < g.Tr;
  const long long li = (long long)bh * g.Tr + i;
  // warm-up: the first W blocks only raise the running max and are streamed again at the end
#ifndef ENTMAX_TAU_WDIV
// warm-up = nkb / WDIV tiles: measured best of {2, 3, 4, 8, 16}: 4 at d = 64, 3 at d = 128 (where the
// MMA share of a tile is larger, so re-streaming is relatively cheaper than transient appends)
#define ENTMAX_TAU_WDIV (D == 128 ? 3 : 4)
#endif
  const int W = nkb >= 32 ? max(4, nkb / (ENTMAX_TAU_WDIV)) : nkb / (ENTMAX_TAU_WDIV);

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar_q, 1);
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kTauSBuf; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&s_empty[s], kTauMathWarps / kTauSBuf);   // the 4 warps of one group
    }
    ptx::mbar_init(&dec_bar, 1);
    ptx::fence_mbar_init();
    s_overflow = 0;
  }
  for (int j = threadIdx.x; j < g.Tc; j += blockDim.x) {
    cflag[j] = 0;
    aflag[j] = 0;
  }
  if (threadIdx.x < kBr) mshare[threadIdx.x] = -INFINITY;
  if (threadIdx.x == 0) ENTMAX_TRACE_EV(8000);
  if (warp == kTauMathWarps + 1) ptx::tmem_alloc<128 * kTauSBuf>(&tmem_base_sh);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();   // the previous kernel (e.g. last step's dQ reading τ) is complete

  if (warp == kTauMathWarps) {
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
      tma_tile<D>(sK + st * C::TILE, &tk, &k_full[st], j * kBc, h, b);
      ++k;
    };
    for (int t = 0; t < nkb + W; ++t) load(t < nkb ? t : t - nkb);
    ptx::mbar_wait(&dec_bar, 0);
    int fb = s_fallback;
    if (fb == 1) {
      for (int j = 0; j < nkb; ++j) load(j);                 // tier 1
      ptx::mbar_wait(&dec_bar, 1);
      fb = s_fallback;
    }
    if (fb == 2)
      for (int t = 0; t < n_iter; ++t)
        for (int j = 0; j < nkb; ++j) load(j);               // tier 2
  } else if (warp == kTauMathWarps + 1) {
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
      ptx::mma_commit_elect(&k_empty[st]);
      ptx::mma_commit_elect(&s_full[sb]);
      ++k;
    };
    for (int p = 0; p < nkb + W; ++p) mma();
    ptx::mbar_wait(&dec_bar, 0);
    int fb = s_fallback;
    if (fb == 1) {
      for (int p = 0; p < nkb; ++p) mma();
      ptx::mbar_wait(&dec_bar, 1);
      fb = s_fallback;
    }
    if (fb == 2)
      for (int p = 0; p < n_iter * nkb; ++p) mma();
  } else {
    // ---------------------------------------------------------------- math warps (512 threads)
    const int tid = threadIdx.x;
    const int r = tid & 127, qc = tid >> 7;
    const int row = i * kBr + r;
    const bool valid = row < g.N;
    const int my_last = g.causal ? row : g.N - 1;
    const int cta_last = g.causal ? i * kBr : g.N - 1;
    // Work split: warp group qc (warps 4qc..4qc+3, one per TMEM lane quadrant) owns S buffer qc and
    // processes every tile whose global stream index k satisfies k % 4 == qc, all 128 columns of it
    // in four 32-column chunks.  The four groups work on four different tiles at once, so the MMA
    // for tile k+4 waits only on group qc, and a warp's per-tile overheads cover 128 columns.
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + qc * 128;
    int kglob = 0;   // global stream index of the next pass's first tile (the MMA issuer's order)
    const uint32_t sfull = ptx::smem_u32(&s_full[qc]), sempty = ptx::smem_u32(&s_empty[qc]);

    auto wait_tile = [&](int kk) {
      if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * (kk >> 2));
      ptx::mbar_wait_addr(sfull, (kk >> 2) & 1);
      if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * (kk >> 2) + 1);
      ptx::tc_fence_after();
    };
    // chunk c (columns 32c .. 32c+31 of key block j) of the waited tile, masked; the last chunk's
    // load releases the S buffer to the MMA issuer
    auto read_chunk = [&](int j, int c, float (&s)[32]) {
      uint32_t ra[32];
#ifdef ENTMAX_TRACE_NOLD
#pragma unroll
      for (int e = 0; e < 32; ++e) ra[e] = 0u;
#else
      ptx::tmem_ld32(lane_base + c * 32, ra);
      ptx::tmem_wait_ld();
#endif
      if (c == 3) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_addr(sempty);
        if (threadIdx.x == 0) ENTMAX_TRACE_EV(3072 + 3 * (j >> 2) + 2);
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) s[e] = __uint_as_float(ra[e]);
      if ((j + 1) * kBc - 1 > cta_last) {
        const int key0 = j * kBc + c * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (key0 + e > my_last) s[e] = -1e30f;   // finite: x + |x| stays exact (no inf − inf)
      }
    };
    // first step t >= 0 of a pass starting at global index k0 that belongs to this group
    auto first_t = [&](int k0) { return (qc - k0 % kTauSBuf + kTauSBuf) % kTauSBuf; };

    // fallback decision of the CTA (s_overflow is read after the barrier: every thread's write to it must
    // be visible): 0 lists complete; 1 rebuild them with the exact threshold (tier 1); 2 stream Alg. 3
    // passes (tier 2) — taken directly when a list is more than twice over its capacity
    auto decide = [&](int use) {
      ptx::named_bar_sync(1, kTauMath);
      if (tid == 0) {
        const int any = s_overflow;
        s_fallback = any == 0 ? 0 : (use == 1 || (any & 2)) ? 2 : 1;
      }
      ptx::named_bar_sync(1, kTauMath);
      return s_fallback != 0;
    };

    // Σ of the row's four fixed-point partial sums (integer adds: exact, any order) → fp32 a0, a1, a2;
    // only the four warps that share the row's TMEM lane quadrant take part (barrier 2 + quadrant)
    // fixed-point units (FxSum): 2^-23 for E != 0; generic α 2^-32 (f, f') and u2 (f'')
    const float u01 = E != 0 ? 8388608.0f : 4294967296.0f;
    const float u2 = E != 0 ? 8388608.0f : (ap.em2 < 0.f ? 1048576.0f : 4294967296.0f);
    auto row_sum3_fx = [&](const FxSum& q, float& a0, float& a1, float& a2) {
      unsigned long long* x64 = reinterpret_cast<unsigned long long*>(xch);
      const uint32_t qbar = 2u + (uint32_t)(warp & 3);
      ptx::named_bar_sync(qbar, 128);
      x64[tid] = q.q0;
      x64[kTauMath + tid] = q.q1;
      x64[2 * kTauMath + tid] = q.q2;
      ptx::named_bar_sync(qbar, 128);
      const unsigned long long s0 = x64[r] + x64[128 + r] + x64[256 + r] + x64[384 + r];
      const unsigned long long s1 =
          x64[kTauMath + r] + x64[kTauMath + 128 + r] + x64[kTauMath + 256 + r] + x64[kTauMath + 384 + r];
      const unsigned long long s2 = x64[2 * kTauMath + r] + x64[2 * kTauMath + 128 + r] +
                                    x64[2 * kTauMath + 256 + r] + x64[2 * kTauMath + 384 + r];
      a0 = (float)s0 * (1.0f / u01);
      a1 = (float)s1 * (1.0f / u01);
      a2 = (float)s2 * (1.0f / u2);
    };

    // this thread's private list: slots [qc·kCapQ, (qc+1)·kCapQ) of row r
    const uint32_t ls0 = ptx::smem_u32(list_s) + (uint32_t)(qc * kCapQ) * 512u + r * 4;
    const uint32_t lj0 = ptx::smem_u32(list_j) + (uint32_t)(qc * kCapQ) * 256u + r * 2;
    const uint32_t ls_end = ls0 + (uint32_t)kCapQ * 512u;
    uint32_t as = ls0, aj = lj0;
    const uint32_t msh = ptx::smem_u32(mshare) + r * 4;
    const uint32_t cflag_s = ptx::smem_u32(cflag);
    const float inv_cp = 1.0f / ap.cp;    // (the 3e-6 margin dwarfs the product's rounding)
    // conservative score threshold: s <= thr(m) ⇒ fma(s, c', −τ_lo(m)) <= 0 (margin >> fma rounding)
    // = m − (1 + margin)/c′ with margin 3e-6·(|m|·c′ + 1.000001) >= the former max(|m·c′ − 1|, 1e-6)·3e-6: two
    // instructions per refresh (FFMA with |m|, FADD), and never above the former threshold
    const float thr_c = inv_cp * (1.0f + 3.0e-6f * 1.000001f);
    auto thr_of = [&](float m) { return valid ? fmaf(fabsf(m), -3.0e-6f, m) - thr_c : INFINITY; };

    // One streaming pass appending the scores above the threshold to the thread's private list.
    // online: the threshold follows the running max of the row (own quarter + the row's published
    // value: a benign race, any value read is a lower bound of m); the first W blocks only raise
    // the max and are appended when they stream again at the end.  !online: fixed threshold `thr`.
    float mrun = -INFINITY, thr = thr_of(-INFINITY);
    constexpr int kChunkUnroll = D == 64 ? 4 : 1;
    auto stream_pass = [&](bool online) {
      const int nsteps = online ? nkb + W : nkb;
      for (int t = first_t(kglob); t < nsteps; t += kTauSBuf) {
        const int j = t < nkb ? t : t - nkb;
        wait_tile(kglob + t);
        // the four chunks of a tile unrolled at d = 64 (config 2 τ −3 %); rolled at d = 128, where the
        // unrolled loop measured 17 % slower
#pragma unroll kChunkUnroll
        for (int c = 0; c < 4; ++c) {
          const float mread = online ? ptx::ld_shared_f32(msh) : 0.f;   // the row's published max
          float s[32];
          read_chunk(j, c, s);
#ifdef ENTMAX_TAU_NOMATH   // diagnostics: streaming floor (TMEM loads only; results invalid)
          if (mread != -12345.f) continue;
#endif
          float gm[4];
#pragma unroll
          for (int gq = 0; gq < 4; ++gq) {
            const float* sg = s + 8 * gq;
            gm[gq] = fmax3(fmax3(sg[0], sg[1], sg[2]), fmax3(sg[3], sg[4], sg[5]), fmaxf(sg[6], sg[7]));
          }
          const float tmax = fmax3(fmaxf(gm[0], gm[1]), gm[2], gm[3]);
          if (online && t < nkb) {
            if (tmax > mread) ptx::st_shared_f32(msh, fmaxf(tmax, mrun));
            mrun = fmax3(mrun, tmax, mread);
            thr = thr_of(mrun);                 // branch-free (same value when mrun is unchanged)
            if (t < W) continue;
          }
          bool hit[4];
#pragma unroll
          for (int gq = 0; gq < 4; ++gq) hit[gq] = gm[gq] > thr;
#ifdef ENTMAX_TAU_NOAPPEND
          if (thr != -12345.f) continue;   // diagnostics: timing of the common path only
#endif
          if (!__any_sync(0xffffffffu, tmax > thr)) continue;   // (= any hit)
          if (lane == 0) ptx::st_shared_u8(cflag_s + j, 1);   // τ_lo candidate block (a superset when online)
          const uint32_t tag = (uint32_t)j;
          // groups of 8 keys with a candidate in some lane: warp-uniform branch.  A lane with one hit
          // in the group appends the group max; the per-key path runs only when some lane's
          // second-largest key of the group is a hit too.
#pragma unroll
          for (int gq = 0; gq < 4; ++gq) {
            if (!__any_sync(0xffffffffu, hit[gq])) continue;
            const float* sg = s + 8 * gq;
            float hh[4], ll[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              hh[q] = fmaxf(sg[2 * q], sg[2 * q + 1]);
              ll[q] = fminf(sg[2 * q], sg[2 * q + 1]);
            }
            const float l01 = fmax3(fminf(hh[0], hh[1]), ll[0], ll[1]),
                        l23 = fmax3(fminf(hh[2], hh[3]), ll[2], ll[3]);
            const float m2 = fmax3(fminf(fmaxf(hh[0], hh[1]), fmaxf(hh[2], hh[3])), l01, l23);
            if (__any_sync(0xffffffffu, m2 > thr)) {
#pragma unroll
              for (int e = 0; e < 8; ++e) list_append(as, aj, ls_end, sg[e], thr, tag);
            } else {
              list_append(as, aj, ls_end, gm[gq], thr, tag);
            }
          }
        }
      }
      kglob += nsteps;
    };
    auto list_len = [&]() { return (int)((as - ls0) >> 9); };

    if (tid == 0) ENTMAX_TRACE_EV(8003);
    stream_pass(true);
    if (tid == 0) ENTMAX_TRACE_EV(8004);
    // row max m (Alg. 1 line 4) and bracket
    xch[tid] = mrun;
    ptx::named_bar_sync(1, kTauMath);
    const float smax = fmax3(fmaxf(xch[r], xch[128 + r]), xch[256 + r], xch[384 + r]);
    const float n_vis = g.causal ? (float)(row + 1) : (float)g.N;
    RowState rs = bracket_init(smax * ap.cp, n_vis, ap.alpha);
    thr = thr_of(smax);
    if (list_len() > kCapQ) {
      // overflow: estimate the exact-threshold list length from the stored entries that pass the
      // final threshold, extrapolated to every hit; if even that exceeds the capacity, a tier-1
      // rebuild would overflow too, so go straight to tier 2
      int above = 0;
      for (int c = 0; c < kCapQ; ++c) above += ptx::ld_shared_f32(ls0 + (uint32_t)c * 512u) > thr ? 1 : 0;
      atomicOr(&s_overflow, above * list_len() > kCapQ * kCapQ ? 3 : 1);
    }
    int* qcnt = reinterpret_cast<int*>(xch) + kTauMath;   // [4][128] list lengths (xch[0..511]: row maxima)
    qcnt[qc * kBr + r] = list_len();
    bool fallback = decide(0);
    if (tid == 0 && s_fallback == 1) ENTMAX_TRACE_COUNT(8100);
    if (tid == 0 && s_fallback == 2) ENTMAX_TRACE_COUNT(8103);
    if (tid == 0) ENTMAX_TRACE_COUNT(8102);
    if (s_fallback == 1) {
      // tier 1: rebuild the lists with the exact threshold
      if (tid == 0) {
        ptx::mbar_arrive(&dec_bar);
        s_overflow = 0;
      }
      as = ls0;
      aj = lj0;
      ptx::named_bar_sync(1, kTauMath);
      stream_pass(false);
      if (list_len() > kCapQ) s_overflow = 1;
      qcnt[qc * kBr + r] = list_len();
      fallback = decide(1);
      if (tid == 0 && fallback) ENTMAX_TRACE_COUNT(8101);
    }

    if (!fallback) {
      // ---- T iterations of Alg. 1 on the row lists: fixed-point sums (FxSum), so τ is bitwise
      // reproducible whichever path produced the lists.  The four quarter lists of a row are summed by
      // four adjacent lanes of one warp (thread → row 8·warp + lane/4, quarter lane % 4), so the row sums
      // are two xor-shuffles per iteration — no block barriers in the iteration loop.
      if (tid == 0) ENTMAX_TRACE_EV(8005);
      const int rr = warp * 8 + (lane >> 2), qq = lane & 3;
      const int rowr = i * kBr + rr;
      const bool validr = rowr < g.N;
      const uint32_t ls0r = ptx::smem_u32(list_s) + (uint32_t)(qq * kCapQ) * 512u + rr * 4;
      const uint32_t lj0r = ptx::smem_u32(list_j) + (uint32_t)(qq * kCapQ) * 256u + rr * 2;
      const int n = qcnt[qq * kBr + rr];
      const float smr = fmax3(fmaxf(xch[rr], xch[128 + rr]), xch[256 + rr], xch[384 + rr]);
      RowState rq = bracket_init(smr * ap.cp, g.causal ? (float)(rowr + 1) : (float)g.N, ap.alpha);
      // the first kReg entries live in registers for all T iterations (−∞ pads contribute zeros)
      constexpr int kReg = 12;
      float lr[kReg];
#pragma unroll
      // (finite pads: the packed sums below form x + |x|)
      for (int c = 0; c < kReg; ++c) lr[c] = c < n ? ptx::ld_shared_f32(ls0r + (uint32_t)c * 512u) : -1e30f;
      for (int t = 0; t < n_iter; ++t) {
        float a0, a1, a2;
        if constexpr (E != 0) {   // <= 4·kCapQ (< 256) terms per row: 32-bit fixed-point sums
          // pairs of entries in packed f32x2 (accum_fx32_pair_raw: bitwise the terms of accum_fx32)
          uint32_t p0 = 0, p1 = 0, p2 = 0;
          const float2 cp2 = make_float2(ap.cp, ap.cp), nt2 = make_float2(-rq.tau, -rq.tau);
#pragma unroll
          for (int c = 0; c < kReg; c += 2)
            accum_fx32_pair_raw<E>(ffma2(make_float2(lr[c], lr[c + 1]), cp2, nt2), p0, p1, p2);
          int nterms = kReg;
#pragma unroll 2
          for (int c = kReg; c < n; c += 2) {
            const float v0 = ptx::ld_shared_f32(ls0r + (uint32_t)c * 512u);
            const float v1 = c + 1 < n ? ptx::ld_shared_f32(ls0r + (uint32_t)(c + 1) * 512u) : -1e30f;
            accum_fx32_pair_raw<E>(ffma2(make_float2(v0, v1), cp2, nt2), p0, p1, p2);
            nterms += 2;
          }
          const uint32_t bias = (uint32_t)nterms * 0x3f800000u;
          p0 -= bias;
          p1 -= bias;
          p2 -= bias;
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            p0 += __shfl_xor_sync(0xffffffffu, p0, o);
            p1 += __shfl_xor_sync(0xffffffffu, p1, o);
            p2 += __shfl_xor_sync(0xffffffffu, p2, o);
          }
          a0 = (float)p0 * (1.0f / u01);
          a1 = (float)p1 * (1.0f / u01);
          a2 = (float)p2 * (1.0f / u2);
        } else {
          FxSum q{0ull, 0ull, 0ull};
#pragma unroll
          for (int c = 0; c < kReg; ++c) {
            const float x = fmaf(lr[c], ap.cp, -rq.tau);
            if (x > 0.f) accum_fx<E>(x, ap, u2, q);
          }
#pragma unroll 4
          for (int c = kReg; c < n; ++c) {
            const float x = fmaf(ptx::ld_shared_f32(ls0r + (uint32_t)c * 512u), ap.cp, -rq.tau);
            if (x > 0.f) accum_fx<E>(x, ap, u2, q);
          }
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            q.q0 += __shfl_xor_sync(0xffffffffu, q.q0, o);
            q.q1 += __shfl_xor_sync(0xffffffffu, q.q1, o);
            q.q2 += __shfl_xor_sync(0xffffffffu, q.q2, o);
          }
          a0 = (float)q.q0 * (1.0f / u01);
          a1 = (float)q.q1 * (1.0f / u01);
          a2 = (float)q.q2 * (1.0f / u2);
        }
        alg1_update(rq, a0, a1, a2, ap);
      }
      if (tid == 0) ENTMAX_TRACE_EV(8008);
      if (validr) {
        if (qq == 0) tau_out[(long long)bh * g.N + rowr] = rq.tau;
        // exact block activity from the final τ (same fma test as the output kernel)
        const uint32_t af = ptx::smem_u32(aflag);
#pragma unroll
        for (int c = 0; c < kReg; ++c)
          if (fmaf(lr[c], ap.cp, -rq.tau) > 0.f) ptx::st_shared_u8(af + ptx::ld_shared_u16(lj0r + (uint32_t)c * 256u), 1);
#pragma unroll 4
        for (int c = kReg; c < n; ++c)
          if (fmaf(ptx::ld_shared_f32(ls0r + (uint32_t)c * 512u), ap.cp, -rq.tau) > 0.f)
            ptx::st_shared_u8(af + ptx::ld_shared_u16(lj0r + (uint32_t)c * 256u), 1);
      }
      if (tid == 0) ENTMAX_TRACE_EV(8009);
      ptx::named_bar_sync(1, kTauMath);
      if (tid == 0) ENTMAX_TRACE_EV(8010);
      if (warp == 0 && real_cta) {
        const int nb = compact_flags(aflag, nkb, cand_idx + li * g.Tc);
        if (lane == 0) cand_cnt[li] = nb;
      }
      if (tid == 0) ENTMAX_TRACE_EV(8011);
      if (tid == 0) {
        __threadfence_block();
        ptx::mbar_arrive(&dec_bar);
      }
    } else {
      // ---- tier 2: streaming Alg. 3 passes over every visible block; the output kernel gets this CTA's
      // τ_lo candidate blocks
      if (warp == 0) {
        if (real_cta) {
          const int nb = compact_flags(cflag, nkb, cand_idx + li * g.Tc);
          if (lane == 0) cand_cnt[li] = nb;
        }
        if (lane == 0) {
          __threadfence_block();
          ptx::mbar_arrive(&dec_bar);
        }
      }
      for (int it = 0; it < n_iter; ++it) {
        FxSum q{0ull, 0ull, 0ull};
        for (int t = first_t(kglob); t < nkb; t += kTauSBuf) {
          wait_tile(kglob + t);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float s[32];
            read_chunk(t, c, s);
            float cm = fmaxf(s[0], s[31]);
#pragma unroll
            for (int e = 1; e < 31; e += 2) cm = fmax3(cm, s[e], s[e + 1]);
            if (__any_sync(0xffffffffu, fmaf(cm, ap.cp, -rs.tau) > 0.f)) {
              if constexpr (E != 0) {   // 32 terms per chunk on pairs in packed f32x2 (accum_fx32_pair_raw)
                uint32_t p0 = 0, p1 = 0, p2 = 0;
                const float2 cp2 = make_float2(ap.cp, ap.cp), nt2 = make_float2(-rs.tau, -rs.tau);
#pragma unroll
                for (int e = 0; e < 32; e += 2)
                  accum_fx32_pair_raw<E>(ffma2(make_float2(s[e], s[e + 1]), cp2, nt2), p0, p1, p2);
                q.q0 += p0 - 32u * 0x3f800000u;   // (mod 2³²: 32 terms of at most 2²³ each)
                q.q1 += p1 - 32u * 0x3f800000u;
                q.q2 += p2 - 32u * 0x3f800000u;
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                  const float x = fmaf(s[e], ap.cp, -rs.tau);
                  if (x > 0.f) accum_fx<E>(x, ap, u2, q);
                }
              }
            }
          }
        }
        kglob += nkb;
        float a0, a1, a2;
        row_sum3_fx(q, a0, a1, a2);
        alg1_update(rs, a0, a1, a2, ap);
      }
      if (qc == 0 && valid) tau_out[(long long)bh * g.N + row] = rs.tau;
    }
  }
  ptx::tc_fence_before();
  if (threadIdx.x == 0) ENTMAX_TRACE_EV(8006);
  __syncthreads();
  if (threadIdx.x == 0) ENTMAX_TRACE_EV(8007);
  if (warp == kTauMathWarps + 1) ptx::tmem_dealloc<128 * kTauSBuf>(tmem);
}

}  // namespace sm100
}  // namespace entmax
