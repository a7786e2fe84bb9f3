// simt_kernels.cuh — FP32-arithmetic SIMT kernels for the whole hot path.
//
// Used for fp32 inputs (config 1 of BASELINE.json needs true-fp32 scores to meet the 1e-4
// bar; tf32 tensor cores give ~5e-3) and for head dims the tcgen05 kernels do
// not cover.  One thread owns one query row (τ, forward output, dQ) or one key row (dK/dV);
// K/V (or Q/dO) tiles are staged in shared memory and read as broadcasts.  Same block
// geometry (B_r = B_c = 128) and the same mask/table semantics as the tcgen05 kernels.
#pragma once

#include "common.cuh"

namespace entmax {
namespace simt {

template <int D>
struct Tile {
  static constexpr int KT = (4096 / D) < 128 ? (4096 / D) : 128;  // rows per staged tile
};

// Stage rows [r0, r0+KT) of a [N,d] head (row stride sn) into smem as fp32, zero past N.
template <typename T, int D>
__device__ __forceinline__ void stage_rows(float (*dst)[D], const T* src, long long sn, int r0, int N) {
  constexpr int KT = Tile<D>::KT;
  for (int idx = threadIdx.x; idx < KT * D; idx += blockDim.x) {
    int rr = idx / D, cc = idx - (idx / D) * D;
    int row = r0 + rr;
    dst[rr][cc] = (row < N) ? to_f<T>(src[(long long)row * sn + cc]) : 0.f;
  }
}

template <int D>
__device__ __forceinline__ float dot_row(const float* a, const float* b) {
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) s = fmaf(a[c], b[c], s);
  return s;
}

// τ per query row: pass 0 = row max, then T passes of Alg. 1 over all visible keys (Alg. 3).
template <typename T, int D, int E>
__global__ void __launch_bounds__(128) tau_kernel(const T* __restrict__ q, const T* __restrict__ k, Geom g,
                                                  AlphaParams ap, int n_iter, float* __restrict__ tau_out) {
  constexpr int KT = Tile<D>::KT;
  __shared__ float ks[KT][D];
  const int i = blockIdx.x, bh = blockIdx.y;
  const int r = i * kBr + threadIdx.x;
  const bool valid = r < g.N;
  const T* qh = q + g.head_off(bh);
  const T* kh = k + g.head_off(bh);
  float qr[D];
#pragma unroll
  for (int c = 0; c < D; ++c) qr[c] = valid ? to_f<T>(qh[(long long)r * g.sn + c]) : 0.f;
  const int kend = g.causal ? min(g.N, (i + 1) * kBr) : g.N;
  const int my_last = g.causal ? r : g.N - 1;

  float smax = -INFINITY;
  for (int kt = 0; kt < kend; kt += KT) {
    __syncthreads();
    stage_rows<T, D>(ks, kh, g.sn, kt, kend);
    __syncthreads();
    const int jn = min(KT, kend - kt);
    for (int j = 0; j < jn; ++j)
      if (kt + j <= my_last) smax = fmaxf(smax, dot_row<D>(qr, ks[j]));
  }
  const float n_vis = g.causal ? (float)(r + 1) : (float)g.N;
  RowState st = bracket_init(smax * ap.cp, n_vis, ap.alpha);
  for (int t = 0; t < n_iter; ++t) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int kt = 0; kt < kend; kt += KT) {
      __syncthreads();
      stage_rows<T, D>(ks, kh, g.sn, kt, kend);
      __syncthreads();
      const int jn = min(KT, kend - kt);
      for (int j = 0; j < jn; ++j) {
        if (kt + j <= my_last) {
          float x = fmaf(dot_row<D>(qr, ks[j]), ap.cp, -st.tau);
          accum_f<E>(x, ap, a0, a1, a2);
        }
      }
    }
    alg1_update(st, a0, a1, a2, ap);
  }
  if (valid) tau_out[(long long)bh * g.N + r] = st.tau;
}

// Output pass over every visible key block; decides M_ij exactly (any x > 0), writes the mask
// row, the 𝒬_i table, O and O⁽²⁾.
template <typename T, int D, int E>
__global__ void __launch_bounds__(128) out_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                  const T* __restrict__ v, Geom g, AlphaParams ap,
                                                  const float* __restrict__ tau, T* __restrict__ o,
                                                  float* __restrict__ o2, uint8_t* __restrict__ mask,
                                                  int32_t* __restrict__ row_cnt, int32_t* __restrict__ row_idx) {
  constexpr int KT = Tile<D>::KT;
  __shared__ float ks[KT][D];
  __shared__ float vs[KT][D];
  const int i = blockIdx.x, bh = blockIdx.y;
  const int r = i * kBr + threadIdx.x;
  const bool valid = r < g.N;
  const long long hoff = g.head_off(bh);
  const T* qh = q + hoff;
  const T* kh = k + hoff;
  const T* vh = v + hoff;
  float qr[D], oa[D], o2a[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    qr[c] = valid ? to_f<T>(qh[(long long)r * g.sn + c]) : 0.f;
    oa[c] = 0.f;
    o2a[c] = 0.f;
  }
  const float tr = valid ? tau[(long long)bh * g.N + r] : 0.f;
  const int my_last = g.causal ? r : g.N - 1;
  const int nkb = g.visible_kblocks(i);
  float usum = 0.f;
  int cnt = 0;
  uint8_t* mrow = mask + ((long long)bh * g.Tr + i) * g.Tc;
  int32_t* lrow = row_idx + ((long long)bh * g.Tr + i) * g.Tc;
  for (int jb = 0; jb < nkb; ++jb) {
    bool act = false;
    for (int kt = jb * kBc; kt < min(g.N, (jb + 1) * kBc); kt += KT) {
      __syncthreads();
      stage_rows<T, D>(ks, kh, g.sn, kt, g.N);
      stage_rows<T, D>(vs, vh, g.sn, kt, g.N);
      __syncthreads();
      const int jn = min(KT, g.N - kt);
      for (int j = 0; j < jn; ++j) {
        if (valid && kt + j <= my_last) {
          float x = fmaf(dot_row<D>(qr, ks[j]), ap.cp, -tr);
          if (x > 0.f) {
            float p, u;
            p_and_u<E>(x, ap, p, u);
            act = true;
            usum += u;
#pragma unroll
            for (int c = 0; c < D; ++c) {
              oa[c] = fmaf(p, vs[j][c], oa[c]);
              o2a[c] = fmaf(u, vs[j][c], o2a[c]);
            }
          }
        }
      }
    }
    const int any = __syncthreads_or(act ? 1 : 0);
    if (threadIdx.x == 0 && mask) {   // (unmasked mode: no mask / table output)
      mrow[jb] = any ? 1 : 0;
      if (any) lrow[cnt++] = jb;
    }
  }
  if (mask) {
    for (int jb = nkb + threadIdx.x; jb < g.Tc; jb += blockDim.x) mrow[jb] = 0;
    if (threadIdx.x == 0) row_cnt[(long long)bh * g.Tr + i] = cnt;
  }
  if (valid) {
    T* orow = o + hoff + (long long)r * g.sn;
#pragma unroll
    for (int c = 0; c < D; ++c) orow[c] = from_f<T>(oa[c]);
    if (o2 != nullptr) {
      float* o2row = o2 + ((long long)bh * g.N + r) * D;   // fp32, contiguous
      const float inv = 1.0f / usum;
#pragma unroll
      for (int c = 0; c < D; ++c) o2row[c] = o2a[c] * inv;
    }
  }
}

// dK_j, dV_j over 𝒦_j (Alg. 4): one thread per key row.
template <typename T, int D, int E>
__global__ void __launch_bounds__(128) dkdv_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                   const T* __restrict__ v, const T* __restrict__ dO, Geom g,
                                                   AlphaParams ap, const float* __restrict__ tau,
                                                   const float* __restrict__ delta,
                                                   const int32_t* __restrict__ col_cnt,
                                                   const int32_t* __restrict__ col_idx, T* __restrict__ dk,
                                                   T* __restrict__ dv) {
  constexpr int KT = Tile<D>::KT;
  __shared__ float qs[KT][D];
  __shared__ float ds_[KT][D];
  __shared__ float ts[KT], dls[KT];
  const int jb = blockIdx.x, bh = blockIdx.y;
  const int key = jb * kBc + threadIdx.x;
  const bool valid = key < g.N;
  const long long hoff = g.head_off(bh);
  float kr[D], vr[D], dka[D], dva[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    kr[c] = valid ? to_f<T>(k[hoff + (long long)key * g.sn + c]) : 0.f;
    vr[c] = valid ? to_f<T>(v[hoff + (long long)key * g.sn + c]) : 0.f;
    dka[c] = 0.f;
    dva[c] = 0.f;
  }
  // unmasked mode (col_idx == nullptr): every query block that sees key block jb
  const int i0 = g.causal ? (jb * kBc) / kBr : 0;
  const int cnt = col_idx ? col_cnt[(long long)bh * g.Tc + jb] : g.Tr - i0;
  const int32_t* lst = col_idx ? col_idx + ((long long)bh * g.Tc + jb) * g.Tr : nullptr;
  for (int t = 0; t < cnt; ++t) {
    const int ib = lst ? lst[t] : i0 + t;
    for (int rt = ib * kBr; rt < min(g.N, (ib + 1) * kBr); rt += KT) {
      __syncthreads();
      stage_rows<T, D>(qs, q + hoff, g.sn, rt, g.N);
      stage_rows<T, D>(ds_, dO + hoff, g.sn, rt, g.N);
      for (int x = threadIdx.x; x < KT; x += blockDim.x) {
        int row = rt + x;
        ts[x] = row < g.N ? tau[(long long)bh * g.N + row] : 0.f;
        dls[x] = row < g.N ? delta[(long long)bh * g.N + row] : 0.f;
      }
      __syncthreads();
      const int rn = min(KT, g.N - rt);
      for (int rr = 0; rr < rn; ++rr) {
        const int row = rt + rr;
        if (valid && (!g.causal || key <= row)) {
          float x = fmaf(dot_row<D>(qs[rr], kr), ap.cp, -ts[rr]);
          if (x > 0.f) {
            float p, u;
            p_and_u<E>(x, ap, p, u);
            float dp = dot_row<D>(ds_[rr], vr);
            float dsv = u * (dp - dls[rr]);
#pragma unroll
            for (int c = 0; c < D; ++c) {
              dva[c] = fmaf(p, ds_[rr][c], dva[c]);
              dka[c] = fmaf(dsv, qs[rr][c], dka[c]);
            }
          }
        }
      }
    }
  }
  if (valid) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      dk[hoff + (long long)key * g.sn + c] = from_f<T>(dka[c] * ap.scale);
      dv[hoff + (long long)key * g.sn + c] = from_f<T>(dva[c]);
    }
  }
}

// dQ_i over 𝒬_i (Alg. 5): one thread per query row.
template <typename T, int D, int E>
__global__ void __launch_bounds__(128) dq_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                 const T* __restrict__ v, const T* __restrict__ dO, Geom g,
                                                 AlphaParams ap, const float* __restrict__ tau,
                                                 const float* __restrict__ delta, const int32_t* __restrict__ row_cnt,
                                                 const int32_t* __restrict__ row_idx, T* __restrict__ dq) {
  constexpr int KT = Tile<D>::KT;
  __shared__ float ks[KT][D];
  __shared__ float vs[KT][D];
  const int ib = blockIdx.x, bh = blockIdx.y;
  const int row = ib * kBr + threadIdx.x;
  const bool valid = row < g.N;
  const long long hoff = g.head_off(bh);
  float qr[D], dor[D], dqa[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    qr[c] = valid ? to_f<T>(q[hoff + (long long)row * g.sn + c]) : 0.f;
    dor[c] = valid ? to_f<T>(dO[hoff + (long long)row * g.sn + c]) : 0.f;
    dqa[c] = 0.f;
  }
  const float tr = valid ? tau[(long long)bh * g.N + row] : 0.f;
  const float dl = valid ? delta[(long long)bh * g.N + row] : 0.f;
  // unmasked mode (row_idx == nullptr): every visible key block
  const int cnt = row_idx ? row_cnt[(long long)bh * g.Tr + ib] : g.visible_kblocks(ib);
  const int32_t* lst = row_idx ? row_idx + ((long long)bh * g.Tr + ib) * g.Tc : nullptr;
  for (int t = 0; t < cnt; ++t) {
    const int jb = lst ? lst[t] : t;
    for (int kt = jb * kBc; kt < min(g.N, (jb + 1) * kBc); kt += KT) {
      __syncthreads();
      stage_rows<T, D>(ks, k + hoff, g.sn, kt, g.N);
      stage_rows<T, D>(vs, v + hoff, g.sn, kt, g.N);
      __syncthreads();
      const int jn = min(KT, g.N - kt);
      for (int j = 0; j < jn; ++j) {
        if (valid && (!g.causal || kt + j <= row)) {
          float x = fmaf(dot_row<D>(qr, ks[j]), ap.cp, -tr);
          if (x > 0.f) {
            float p, u;
            p_and_u<E>(x, ap, p, u);
            float dp = dot_row<D>(dor, vs[j]);
            float dsv = u * (dp - dl);
#pragma unroll
            for (int c = 0; c < D; ++c) dqa[c] = fmaf(dsv, ks[j][c], dqa[c]);
          }
        }
      }
    }
  }
  if (valid) {
#pragma unroll
    for (int c = 0; c < D; ++c) dq[hoff + (long long)row * g.sn + c] = from_f<T>(dqa[c] * ap.scale);
  }
}

}  // namespace simt

// ---------------------------------------------------------------------------------------
// Kernels shared by both implementations
// ---------------------------------------------------------------------------------------

// δ_i = dO_iᵀ O⁽²⁾_i, fp32 accumulation.  HBM-bound: TPR = d/8 threads per row, each
// reading 8 consecutive elements of dO (one 16-byte vector for bf16) and of O⁽²⁾ (two float4), then a
// TPR-lane shuffle reduction; 256 / TPR rows per 256-thread block.
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <typename T, int TPR>
__global__ void __launch_bounds__(256) delta_kernel(const T* __restrict__ dO, const float* __restrict__ o2,
                                                    const float* __restrict__ tau, Geom g, float* __restrict__ delta,
                                                    float* __restrict__ td) {
  // δ_i = dO_i · O⁽²⁾_i.  With td != NULL (tcgen05 path) also the per-query-block staging array
  // td[bh][i] = {τ of the block's 128 rows | δ of them} (1 KB, +∞ / 0 past N) that the dK/dV kernel's
  // producer pulls with one bulk copy per query block; rows run over the padded T_r·128 rows per head.
  // Padding rows get τ = 1e10 (finite: x = c′s − τ then gives exact zeros through x + |x|) and δ = 0.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // (launched with PDL: see runtime.h)
  const long long prow = ((long long)blockIdx.x * 256 + threadIdx.x) / TPR;
  const int sub = threadIdx.x % TPR;
  const long long rows_pad = (long long)g.B * g.H * g.Tr * kBr;
  const bool in = prow < rows_pad;
  const int bh = in ? (int)(prow / ((long long)g.Tr * kBr)) : 0;
  const int r = in ? (int)(prow - (long long)bh * g.Tr * kBr) : 0;
  const bool ok = in && r < g.N;
  float s = 0.f;
  if (ok) {
    float a[8], b[8];
    load8<T>(dO + g.head_off(bh) + (long long)r * g.sn + sub * 8, a);
    load8<float>(o2 + ((long long)bh * g.N + r) * g.d + sub * 8, b);   // fp32 contiguous [B,H,N,d]
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(a[e], b[e], s);
  }
#pragma unroll
  for (int m = TPR / 2; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if (in && sub == 0) {
    if (ok) delta[(long long)bh * g.N + r] = s;
    if (td != nullptr) {
      float* blk = td + ((long long)bh * g.Tr + r / kBr) * (2 * kBr);
      blk[r % kBr] = ok ? tau[(long long)bh * g.N + r] : 1e10f;   // (finite: see sm100_fb.cuh kPadTau)
      blk[kBr + r % kBr] = ok ? s : 0.f;
    }
  }
}

// 𝒦_j = {i | M_ij = 1} from the mask, increasing i; one thread per (head, j).
__global__ void col_lists_kernel(const uint8_t* __restrict__ mask, int BH, int Tr, int Tc,
                                 int32_t* __restrict__ col_cnt, int32_t* __restrict__ col_idx) {
  // one warp per (head, key block j): the lanes read 32 rows of the column at once and a ballot
  // compacts them in increasing i (the thread-per-column loop was a chain of dependent loads)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // (launched with PDL: see runtime.h)
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)BH * Tc) return;
  const int bh = (int)(w / Tc), j = (int)(w - (long long)(w / Tc) * Tc);
  const uint8_t* m = mask + (long long)bh * Tr * Tc + j;
  int32_t* out = col_idx + ((long long)bh * Tc + j) * Tr;
  int cnt = 0;
  for (int i0 = 0; i0 < Tr; i0 += 32) {
    const int i = i0 + lane;
    const bool f = i < Tr && m[(long long)i * Tc] != 0;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (f) out[cnt + __popc(b & ((1u << lane) - 1u))] = i;
    cnt += __popc(b);
  }
  if (lane == 0) col_cnt[w] = cnt;
}

// bit-packed mask: one thread per output word (32 mask bytes)
__global__ void pack_mask_kernel(const uint8_t* __restrict__ mask, long long rows, int Tc, int words,
                                 uint32_t* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * words) return;
  const long long r = t / words;
  const int w = (int)(t - r * words);
  const uint8_t* m = mask + r * Tc + w * 32;
  const int nb = min(32, Tc - w * 32);
  uint32_t v = 0;
  for (int b = 0; b < nb; ++b) v |= (m[b] != 0 ? 1u : 0u) << b;
  out[t] = v;
}

}  // namespace entmax
