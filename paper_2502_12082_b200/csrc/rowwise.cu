// rowwise.cu — standalone row-wise α-entmax (include/entmax_rowwise.h).
//
// Paper: Alg. 1 on the rows of a matrix, the solver the paper benchmarks on its own
// (n = 8192 Gaussian rows, T = 3); backward = the sparse Jacobian of P:L371-377.
//
// B200 design: the op is HBM-bound (T + 2 reductions over a row that is read once and written
// once), so each row lives in registers for the whole solve: one CTA per row, NT threads × VPT
// values, 16-byte coalesced loads/stores (chunk c of thread t covers elements [(c·NT + t)·W, +W)).
// HBM traffic is exactly one read of s and one write of p (+4 bytes of τ) per row; the Alg. 1
// iterations run over the row's candidates (z > m − 1, compacted into shared memory) plus a
// deterministic block reduction (fixed warp-shuffle tree, then the warp partials in warp order), so
// results are bitwise reproducible.
// Rows longer than NT·VPT (n > 16384) take a streaming variant that re-reads the row from global
// memory (L2) on every pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "entmax_rowwise.h"
#include "common.cuh"
#include "runtime.h"

namespace entmax {
namespace rowwise {

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

template <typename T>
struct Chunk;   // one 16-byte vector
template <>
struct Chunk<float> {
  static constexpr int W = 4;
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Chunk<__nv_bfloat16> {
  static constexpr int W = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// Load chunk `c0` (element offset) of a row into v; entries at or past n get `fill`.
template <typename T>
__device__ __forceinline__ void load_chunk(const T* row, int c0, int n, float fill, float (&v)[Chunk<T>::W]) {
  constexpr int W = Chunk<T>::W;
  if (c0 + W <= n) {
    Chunk<T>::load(row + c0, v);
  } else {
#pragma unroll
    for (int e = 0; e < W; ++e) v[e] = (c0 + e < n) ? to_f<T>(row[c0 + e]) : fill;
  }
}

template <typename T>
__device__ __forceinline__ void store_chunk(T* row, int c0, int n, const float (&v)[Chunk<T>::W]) {
  constexpr int W = Chunk<T>::W;
  if (c0 + W <= n) {
    Chunk<T>::store(row + c0, v);
  } else {
#pragma unroll
    for (int e = 0; e < W; ++e)
      if (c0 + e < n) row[c0 + e] = from_f<T>(v[e]);
  }
}

// Deterministic block reductions.  `red` holds two buffers of [K][NT/32] floats used alternately
// (parity `ph`), so one __syncthreads per reduction suffices: a buffer is rewritten only after
// every thread has passed the next reduction's barrier, i.e. finished reading it.
template <int NT>
__device__ __forceinline__ float block_max(float v, float* red, int& ph) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  float* buf = red + (ph & 1) * 3 * NW;
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
  __syncthreads();
  ++ph;
  float r = buf[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r = fmaxf(r, buf[w]);
  return r;
}

template <int NT>
__device__ __forceinline__ void block_sum3(float& a0, float& a1, float& a2, float* red, int& ph) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  float* buf = red + (ph & 1) * 3 * NW;
  if ((threadIdx.x & 31) == 0) {
    buf[threadIdx.x >> 5] = a0;
    buf[NW + (threadIdx.x >> 5)] = a1;
    buf[2 * NW + (threadIdx.x >> 5)] = a2;
  }
  __syncthreads();
  ++ph;
  a0 = buf[0];
  a1 = buf[NW];
  a2 = buf[2 * NW];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    a0 += buf[w];
    a1 += buf[NW + w];
    a2 += buf[2 * NW + w];
  }
}

// Eq. 4 only (halley = 0): bracket update, τ = midpoint (tie f = 0 → τ_lo, reading c5).
__device__ __forceinline__ void bisect_update(RowState& s, float a0) {
  if (a0 - 1.0f < 0.f) s.hi = s.tau; else s.lo = s.tau;
  s.tau = 0.5f * (s.lo + s.hi);
}

__device__ __forceinline__ void solver_step(RowState& rs, float a0, float a1, float a2, const AlphaParams& ap,
                                            bool halley) {
  if (halley) alg1_update(rs, a0, a1, a2, ap);
  else bisect_update(rs, a0);
}

// u = p^{2−α} (0 off the support): E = 1 → 1[p>0], 2 → √p, 4 → p^{3/4}, generic exp2/log2.
template <int E>
__device__ __forceinline__ float u_of_p(float p, const AlphaParams& ap) {
  if (E == 1) return p > 0.f ? 1.f : 0.f;
  if (E == 2) return sqrtf(fmaxf(p, 0.f));
  if (E == 4) {
    const float r = sqrtf(fmaxf(p, 0.f));
    return r * sqrtf(r);
  }
  return p > 0.f ? exp2f((2.0f - ap.alpha) * __log2f(p)) : 0.f;
}

// L2 prefetch of the row a later CTA will solve (1-D bulk prefetch, one instruction for the whole row;
// `bytes` a multiple of 16).  The register kernels issue their row's loads only when the CTA starts,
// so HBM traffic in flight is bounded by the resident CTAs; a CTA starting on a row that is already in
// L2 finishes sooner.
__device__ __forceinline__ void prefetch_row_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ------------------------------------------------------------------------- register-resident rows
template <typename T, int NT, int VPT, int E>
__global__ void __launch_bounds__(NT) fwd_reg_kernel(const T* s, int n, long long ld, AlphaParams ap,
                                                     int n_iter, int halley, bool compact, T* p,
                                                     float* __restrict__ tau, int pf) {
  constexpr int W = Chunk<T>::W, NC = VPT / W;
  __shared__ float red[2 * 3 * (NT / 32)];
  int ph = 0;
  const long long row = blockIdx.x;
  if (pf && threadIdx.x == 0 && row + pf < gridDim.x)
    prefetch_row_l2(s + (row + pf) * ld, ((uint32_t)n * (uint32_t)sizeof(T)) & ~15u);
  const T* srow = s + row * ld;
  float z[VPT];
  // Alg. 1 line 3: z = (α−1)·s; line 4: m = max z (padding entries past n: a huge finite negative value,
  // so they contribute exact zeros — also to the packed sums below, where x + |x| must not meet ∞ − ∞)
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float v[W];
    load_chunk<T>(srow, (c * NT + threadIdx.x) * W, n, -1e30f, v);
#pragma unroll
    for (int e = 0; e < W; ++e) z[c * W + e] = v[e] * ap.cp;
  }
  float m = z[0];
#pragma unroll
  for (int i = 1; i + 1 < VPT; i += 2) m = fmax3(m, z[i], z[i + 1]);
  if constexpr (VPT % 2 == 0) m = fmaxf(m, z[VPT - 1]);
  m = block_max<NT>(m, red, ph);
  RowState rs = bracket_init(m, (float)n, ap.alpha);   // lines 5-6
  // Candidates (readings c3/c7): every iterate is >= τ_lo = m − 1, so z <= τ_lo gives x = z − τ <= 0
  // (fp32 subtraction is monotone) and an exact zero in f, f′, f″.  The T iterations therefore sum a
  // compacted list of the z > τ_lo in shared memory, ordered by thread and register index through a
  // block-wide exclusive scan of the per-thread counts — deterministic sums, ~3 % of n for Gaussian
  // rows at α = 1.5.
  // (Only for many iterations, compact = n_iter > 4: at T = 3 the register passes are cheaper than
  // the scan's two extra barriers.)
  extern __shared__ float cand[];     // NT·VPT floats when compact: any count fits
  __shared__ int wsum[NT / 32];
  if (!compact) {
    for (int t = 0; t < n_iter; ++t) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f;
      if constexpr (E == 1 || E == 2 || E == 4) {
        // packed f32x2 sums over pairs of values (sm_100a FADD2 / FFMA2 / FMUL2), in doubled units
        // r = x + |x| = 2·x₊ (exact), rescaled by exact powers of two at the end
        float2 A0 = make_float2(0.f, 0.f), A1 = A0, A2 = A0;
        const float2 nt = make_float2(-rs.tau, -rs.tau);
#pragma unroll
        for (int i = 0; i < VPT; i += 2) {
          const float2 x = fadd2(make_float2(z[i], z[i + 1]), nt);
          const float2 r = fadd2(x, fabs2(x));
          if constexpr (E == 1) {          // f = Σx₊ − 1, f' ∝ Σ[x > 0]
            A0 = fadd2(A0, r);
            A1 = fadd2(A1, make_float2(fminf(r.x * 0x1p100f, 1.f), fminf(r.y * 0x1p100f, 1.f)));
          } else if constexpr (E == 2) {   // Σx₊², Σx₊, Σ[x > 0]
            A0 = ffma2(r, r, A0);
            A1 = fadd2(A1, r);
            A2 = fadd2(A2, make_float2(fminf(r.x * 0x1p100f, 1.f), fminf(r.y * 0x1p100f, 1.f)));
          } else {                         // Σx₊⁴, Σx₊³, Σx₊²
            const float2 r2 = fmul2(r, r);
            A0 = ffma2(r2, r2, A0);
            A1 = ffma2(r2, r, A1);
            A2 = fadd2(A2, r2);
          }
        }
        if constexpr (E == 1) {
          a0 = (A0.x + A0.y) * 0.5f;
          a1 = A1.x + A1.y;
        } else if constexpr (E == 2) {
          a0 = (A0.x + A0.y) * 0.25f;
          a1 = (A1.x + A1.y) * 0.5f;
          a2 = A2.x + A2.y;
        } else {
          a0 = (A0.x + A0.y) * 0.0625f;
          a1 = (A1.x + A1.y) * 0.125f;
          a2 = (A2.x + A2.y) * 0.25f;
        }
      } else {
#pragma unroll
        for (int i = 0; i < VPT; ++i) accum_f<E>(z[i] - rs.tau, ap, a0, a1, a2);
      }
      block_sum3<NT>(a0, a1, a2, red, ph);
      solver_step(rs, a0, a1, a2, ap, halley);
    }
  } else {
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < VPT; ++i) cnt += z[i] > rs.lo ? 1 : 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int off = incl - cnt, total = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const int v = wsum[w];
    off += w < wid ? v : 0;
    total += v;
  }
#pragma unroll
  for (int i = 0; i < VPT; ++i)
    if (z[i] > rs.lo) cand[off++] = z[i];
  __syncthreads();
  for (int t = 0; t < n_iter; ++t) {                     // lines 7-14
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int c = threadIdx.x; c < total; c += NT) accum_f<E>(cand[c] - rs.tau, ap, a0, a1, a2);
    block_sum3<NT>(a0, a1, a2, red, ph);
    solver_step(rs, a0, a1, a2, ap, halley);
  }
  }
  // line 15: p = [z − τ]_+^{1/(α−1)}
  T* prow = p + row * ld;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float v[W];
    if constexpr (E == 2) {   // p = x₊² = (r/2)², r = x + |x|: packed, exact
      const float2 nt = make_float2(-rs.tau, -rs.tau);
#pragma unroll
      for (int e = 0; e < W; e += 2) {
        const float2 x = fadd2(make_float2(z[c * W + e], z[c * W + e + 1]), nt);
        const float2 h = fmul2(fadd2(x, fabs2(x)), make_float2(0.5f, 0.5f));
        const float2 pp = fmul2(h, h);
        v[e] = pp.x;
        v[e + 1] = pp.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < W; ++e) {
        float pu, uu;
        p_and_u<E>(z[c * W + e] - rs.tau, ap, pu, uu);
        v[e] = pu;
      }
    }
    store_chunk<T>(prow, (c * NT + threadIdx.x) * W, n, v);
  }
  if (tau && threadIdx.x == 0) tau[row] = rs.tau;
}

template <typename T, int NT, int VPT, int E>
__global__ void __launch_bounds__(NT) bwd_reg_kernel(const T* p, const T* dp, int n,
                                                     long long ld, AlphaParams ap, T* ds, int pf) {
  constexpr int W = Chunk<T>::W, NC = VPT / W;
  __shared__ float red[2 * 3 * (NT / 32)];
  int ph = 0;
  const long long row = blockIdx.x;
  if (pf && threadIdx.x < 2 && row + pf < gridDim.x)
    prefetch_row_l2((threadIdx.x ? dp : p) + (row + pf) * ld, ((uint32_t)n * (uint32_t)sizeof(T)) & ~15u);
  float u[VPT], g[VPT];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float pv[W], gv[W];
    load_chunk<T>(p + row * ld, (c * NT + threadIdx.x) * W, n, 0.f, pv);
    load_chunk<T>(dp + row * ld, (c * NT + threadIdx.x) * W, n, 0.f, gv);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      u[c * W + e] = u_of_p<E>(pv[e], ap);
      g[c * W + e] = gv[e];
    }
  }
  float su = 0.f, sud = 0.f, unused = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    su += u[i];
    sud = fmaf(u[i], g[i], sud);
  }
  block_sum3<NT>(su, sud, unused, red, ph);
  const float r = sud / su;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float v[W];
#pragma unroll
    for (int e = 0; e < W; ++e) v[e] = u[c * W + e] * (g[c * W + e] - r);
    store_chunk<T>(ds + row * ld, (c * NT + threadIdx.x) * W, n, v);
  }
}

// ------------------------------------------------------------------------- streaming (long rows)
constexpr int kStreamNT = 1024;

template <typename T, int E>
__global__ void __launch_bounds__(kStreamNT) fwd_stream_kernel(const T* s, int n, long long ld,
                                                               AlphaParams ap, int n_iter, int halley, T* p,
                                                               float* __restrict__ tau) {
  constexpr int W = Chunk<T>::W, NT = kStreamNT;
  __shared__ float red[2 * 3 * (NT / 32)];
  int ph = 0;
  const long long row = blockIdx.x;
  const T* srow = s + row * ld;
  float m = -INFINITY;
  for (int c0 = threadIdx.x * W; c0 < n; c0 += NT * W) {
    float v[W];
    load_chunk<T>(srow, c0, n, -INFINITY, v);
#pragma unroll
    for (int e = 0; e < W; ++e) m = fmaxf(m, v[e] * ap.cp);
  }
  m = block_max<NT>(m, red, ph);
  RowState rs = bracket_init(m, (float)n, ap.alpha);
  for (int t = 0; t < n_iter; ++t) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int c0 = threadIdx.x * W; c0 < n; c0 += NT * W) {
      float v[W];
      load_chunk<T>(srow, c0, n, -INFINITY, v);
#pragma unroll
      for (int e = 0; e < W; ++e) accum_f<E>(v[e] * ap.cp - rs.tau, ap, a0, a1, a2);
    }
    block_sum3<NT>(a0, a1, a2, red, ph);
    solver_step(rs, a0, a1, a2, ap, halley);
  }
  // in-place safety: every thread has finished reading the row (the last barrier) before any write
  __syncthreads();
  T* prow = p + row * ld;
  for (int c0 = threadIdx.x * W; c0 < n; c0 += NT * W) {
    float v[W];
    load_chunk<T>(srow, c0, n, -INFINITY, v);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      float pu, uu;
      p_and_u<E>(v[e] * ap.cp - rs.tau, ap, pu, uu);
      v[e] = pu;
    }
    store_chunk<T>(prow, c0, n, v);
  }
  if (tau && threadIdx.x == 0) tau[row] = rs.tau;
}

template <typename T, int E>
__global__ void __launch_bounds__(kStreamNT) bwd_stream_kernel(const T* p, const T* dp,
                                                               int n, long long ld, AlphaParams ap, T* ds) {
  constexpr int W = Chunk<T>::W, NT = kStreamNT;
  __shared__ float red[2 * 3 * (NT / 32)];
  int ph = 0;
  const long long row = blockIdx.x;
  float su = 0.f, sud = 0.f, unused = 0.f;
  for (int c0 = threadIdx.x * W; c0 < n; c0 += NT * W) {
    float pv[W], gv[W];
    load_chunk<T>(p + row * ld, c0, n, 0.f, pv);
    load_chunk<T>(dp + row * ld, c0, n, 0.f, gv);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const float u = u_of_p<E>(pv[e], ap);
      su += u;
      sud = fmaf(u, gv[e], sud);
    }
  }
  block_sum3<NT>(su, sud, unused, red, ph);
  const float r = sud / su;
  __syncthreads();
  for (int c0 = threadIdx.x * W; c0 < n; c0 += NT * W) {
    float pv[W], gv[W];
    load_chunk<T>(p + row * ld, c0, n, 0.f, pv);
    load_chunk<T>(dp + row * ld, c0, n, 0.f, gv);
#pragma unroll
    for (int e = 0; e < W; ++e) pv[e] = u_of_p<E>(pv[e], ap) * (gv[e] - r);
    store_chunk<T>(ds + row * ld, c0, n, pv);
  }
}

// ------------------------------------------------------------------------- dispatch
// Prefetch distance of the register kernels: the resident CTAs of the whole GPU (the row the CTA that
// replaces this one will solve), times ENTMAX_RW_PF (diagnostics; 0 disables).
inline int pf_factor() {
  static const int f = [] {
    const char* e = std::getenv("ENTMAX_RW_PF");
    return e ? std::atoi(e) : 1;
  }();
  return f;
}
template <auto Kern>
int pf_distance(int nt, size_t smem) {
  static int resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, Kern, nt, smem) != cudaSuccess) per_sm = 1;
    resident = std::max(1, per_sm) * sms;
  }
  return resident * pf_factor();
}
// Register-path shapes (NT threads × VPT values): chosen by n so a CTA holds its whole row.
template <typename T, int E, typename Op>
int by_n(int n, Op&& op) {
  // (NT, VPT) measured on 8192 × {4096, 8192, 16384} rows: few threads per row (cheap block
  // reductions) with 32 values each for fp32, 64 for bf16 (same bytes per thread); longer rows take
  // more threads, then the streaming variant
  constexpr int W = Chunk<T>::W;
  if (n <= 128 * 2 * W) return op.template run<128, 2 * W>();
  if (n <= 128 * 32) return op.template run<128, 32>();
  if constexpr (W == 8) {
    if (n <= 128 * 64) return op.template run<128, 64>();
    if (n <= 256 * 64) return op.template run<256, 64>();
  } else {
    if (n <= 256 * 32) return op.template run<256, 32>();
    if (n <= 512 * 32) return op.template run<512, 32>();
  }
  return op.template run<0, 0>();   // streaming
}

template <typename T, int E>
struct FwdLaunch {
  const T* s; long long rows; int n; long long ld; AlphaParams ap; int n_iter, halley; T* p; float* tau;
  cudaStream_t st;
  template <int NT, int VPT>
  int run() {
    if constexpr (NT == 0) {
      ProfScope ps("rowwise_fwd_stream", st);
      fwd_stream_kernel<T, E><<<(unsigned)rows, kStreamNT, 0, st>>>(s, n, ld, ap, n_iter, halley, p, tau);
    } else {
      constexpr int smem = NT * VPT * (int)sizeof(float);
      static bool attr = [] {
        return cudaFuncSetAttribute(fwd_reg_kernel<T, NT, VPT, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem) == cudaSuccess;
      }();
      (void)attr;
      ProfScope ps("rowwise_fwd", st);
      const bool compact = n_iter > 4;
      fwd_reg_kernel<T, NT, VPT, E><<<(unsigned)rows, NT, compact ? smem : 0, st>>>(s, n, ld, ap, n_iter, halley,
                                                                                  compact, p, tau,
                                                                                  pf_distance<fwd_reg_kernel<T, NT, VPT, E>>(NT, compact ? smem : 0));
    }
    return cuda_status("entmax_rowwise_fwd");
  }
};

template <typename T, int E>
struct BwdLaunch {
  const T *p, *dp; long long rows; int n; long long ld; AlphaParams ap; T* ds; cudaStream_t st;
  template <int NT, int VPT>
  int run() {
    if constexpr (NT == 0) {
      ProfScope ps("rowwise_bwd_stream", st);
      bwd_stream_kernel<T, E><<<(unsigned)rows, kStreamNT, 0, st>>>(p, dp, n, ld, ap, ds);
    } else {
      ProfScope ps("rowwise_bwd", st);
      bwd_reg_kernel<T, NT, VPT, E><<<(unsigned)rows, NT, 0, st>>>(p, dp, n, ld, ap, ds,
                                                                pf_distance<bwd_reg_kernel<T, NT, VPT, E>>(NT, 0));
    }
    return cuda_status("entmax_rowwise_bwd");
  }
};

// Backward shapes: only two reductions and no iterations, so rows are split over more threads (fewer
// registers per thread, more warps in flight for the HBM stream).
template <typename T, int E, typename Op>
int by_n_bwd(int n, Op&& op) {
  constexpr int W = Chunk<T>::W;
  if (n <= 128 * 2 * W) return op.template run<128, 2 * W>();
  if (n <= 1024 * W) return op.template run<1024, W>();
  if (n <= 1024 * 2 * W) return op.template run<1024, 2 * W>();
  if (n <= 1024 * 16) return op.template run<1024, 16>();   // (<= 64 registers at 1024 threads)
  return op.template run<0, 0>();   // streaming
}

template <template <typename, int> class L, typename T, bool BWD, typename... A>
int by_e(int ecode, int n, A... a) {
  auto go = [n](auto&& op) {
    using Op = std::decay_t<decltype(op)>;
    if constexpr (BWD) return by_n_bwd<T, 0>(n, op);
    else return by_n<T, 0>(n, op);
    (void)sizeof(Op);
  };
  switch (ecode) {
    case 1: return go(L<T, 1>{a...});
    case 2: return go(L<T, 2>{a...});
    case 4: return go(L<T, 4>{a...});
    default: return go(L<T, 0>{a...});
  }
}

int check_common(const void* a, const void* b, long long rows, int n, long long ld, int dtype) {
  if (dtype != ENTMAX_BF16 && dtype != ENTMAX_FP32) return fail(ENTMAX_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (rows < 1 || n < 1) return fail(ENTMAX_ERR_INVALID_ARG, "rows and n must be >= 1 (got %lld, %d)", rows, n);
  if (rows > 0x7fffffffLL) return fail(ENTMAX_ERR_UNSUPPORTED, "rows > 2^31-1 not supported");
  if (ld < n) return fail(ENTMAX_ERR_INVALID_ARG, "ld (%lld) < n (%d)", ld, n);
  const int esz = dtype == ENTMAX_BF16 ? 2 : 4;
  if ((ld * esz) % 16) return fail(ENTMAX_ERR_INVALID_ARG, "ld must be a multiple of 16 bytes");
  if (!a || !b) return fail(ENTMAX_ERR_INVALID_ARG, "NULL tensor pointer");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u)
    return fail(ENTMAX_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  return ENTMAX_OK;
}

int check_alpha_rw(float alpha) {
  if (!(alpha >= 1.001f)) return fail(ENTMAX_ERR_INVALID_ARG, "alpha must be >= 1 + 1e-3 (got %g)", alpha);
  if (alpha > 2.0f) return fail(ENTMAX_ERR_UNSUPPORTED, "alpha > 2 not supported (got %g)", alpha);
  return ENTMAX_OK;
}

}  // namespace rowwise
}  // namespace entmax

using namespace entmax;
using namespace entmax::rowwise;

extern "C" int entmax_rowwise_fwd(const void* s, int64_t rows, int32_t n, int64_t ld, int dtype, float alpha,
                                  int n_iter, int halley, void* p, float* tau, void* stream) {
  int st = check_common(s, p, rows, n, ld, dtype);
  if (st) return st;
  if ((st = check_alpha_rw(alpha))) return st;
  if (n_iter < 1) return fail(ENTMAX_ERR_INVALID_ARG, "n_iter must be >= 1 (got %d)", n_iter);
  if (tau && (reinterpret_cast<uintptr_t>(tau) & 3u)) return fail(ENTMAX_ERR_INVALID_ARG, "tau misaligned");
  const AlphaParams ap = make_alpha_params(alpha, 1.0f);   // z = (α−1)·s (Alg. 1 line 3)
  const int ec = exponent_code(alpha);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const int hb = halley ? 1 : 0;
  if (dtype == ENTMAX_FP32)
    return by_e<FwdLaunch, float, false>(ec, n, static_cast<const float*>(s), (long long)rows, (int)n, (long long)ld, ap,
                                  n_iter, hb, static_cast<float*>(p), tau, cs);
  return by_e<FwdLaunch, __nv_bfloat16, false>(ec, n, static_cast<const __nv_bfloat16*>(s), (long long)rows, (int)n,
                                        (long long)ld, ap, n_iter, hb, static_cast<__nv_bfloat16*>(p), tau, cs);
}

extern "C" int entmax_rowwise_bwd(const void* p, const void* dp, int64_t rows, int32_t n, int64_t ld, int dtype,
                                  float alpha, void* ds, void* stream) {
  int st = check_common(p, dp, rows, n, ld, dtype);
  if (st) return st;
  if ((st = check_common(ds, ds, rows, n, ld, dtype))) return st;
  if ((st = check_alpha_rw(alpha))) return st;
  const AlphaParams ap = make_alpha_params(alpha, 1.0f);
  const int ec = exponent_code(alpha);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  if (dtype == ENTMAX_FP32)
    return by_e<BwdLaunch, float, true>(ec, n, static_cast<const float*>(p), static_cast<const float*>(dp),
                                  (long long)rows, (int)n, (long long)ld, ap, static_cast<float*>(ds), cs);
  return by_e<BwdLaunch, __nv_bfloat16, true>(ec, n, static_cast<const __nv_bfloat16*>(p),
                                        static_cast<const __nv_bfloat16*>(dp), (long long)rows, (int)n,
                                        (long long)ld, ap, static_cast<__nv_bfloat16*>(ds), cs);
}
