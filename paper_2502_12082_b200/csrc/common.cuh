// common.cuh — per-element α-entmax arithmetic and the Alg. 1 row update, shared by the
// SIMT and the tcgen05 kernels of this library (never by the oracle).
//
// Exponent e = 1/(α−1).  The three α of the paper's configs give integer e:
//   α = 2    → e = 1 (sparsemax),  α = 1.5 → e = 2,  α = 1.25 → e = 4.
// They are compile-time specialisations (E = 1, 2, 4); E = 0 is the generic-α path that uses
// exp2/log2.  All arithmetic is fp32.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace entmax {

constexpr int kBr = 128;  // query rows per block  (mask granularity B_r)
constexpr int kBc = 128;  // keys per block         (mask granularity B_c)

struct AlphaParams {
  float alpha;   // α
  float e;       // 1/(α−1)
  float em1;     // e − 1   (= (2−α)/(α−1); exponent of U = P^{2−α})
  float em2;     // e − 2
  float c1;      // −e               (f' = c1 · Σ[x]_+^{e−1},  Eq. 6)
  float c2;      // (2−α)/(α−1)²     (f'' = c2 · Σ[x]_+^{e−2}, Eq. 7)
  float cp;      // (α−1)·scale: z = cp · s_raw  (Alg. 1 line 3 with Eq. 1 scale)
  float scale;   // c = 1/√d or user value
};

inline AlphaParams make_alpha_params(float alpha, float scale) {
  AlphaParams a;
  a.alpha = alpha;
  a.e = 1.0f / (alpha - 1.0f);
  a.em1 = a.e - 1.0f;
  a.em2 = a.e - 2.0f;
  a.c1 = -a.e;
  a.c2 = (2.0f - alpha) / ((alpha - 1.0f) * (alpha - 1.0f));
  a.cp = (alpha - 1.0f) * scale;
  a.scale = scale;
  return a;
}

// Exponent code dispatched at launch: 1, 2, 4 or 0 (generic).
inline int exponent_code(float alpha) {
  if (alpha == 2.0f) return 1;
  if (alpha == 1.5f) return 2;
  if (alpha == 1.25f) return 4;
  return 0;
}

__device__ __forceinline__ float gpow(float x, float p) {  // x > 0
  return exp2f(p * __log2f(x));
}

// Accumulate the three sums of Eq. 3 / Eq. 6 / Eq. 7 for one element x = z − τ:
//   a0 += [x]_+^e,  a1 += [x]_+^{e−1},  a2 += [x]_+^{e−2}   ([x]_+^p := 0 for x <= 0, reading c7)
template <int E>
__device__ __forceinline__ void accum_f(float x, const AlphaParams& ap, float& a0, float& a1, float& a2) {
  if (E == 1) {
    float xp = fmaxf(x, 0.f);
    a0 += xp;
    a1 += (x > 0.f) ? 1.f : 0.f;
  } else if (E == 2) {
    float xp = fmaxf(x, 0.f);
    a0 = fmaf(xp, xp, a0);
    a1 += xp;
    a2 += (x > 0.f) ? 1.f : 0.f;
  } else if (E == 4) {
    float xp = fmaxf(x, 0.f);
    float x2 = xp * xp;
    a0 = fmaf(x2, x2, a0);
    a1 = fmaf(x2, xp, a1);
    a2 += x2;
  } else {
    if (x > 0.f) {
      float l = __log2f(x);
      a0 += exp2f(ap.e * l);
      a1 += exp2f(ap.em1 * l);
      a2 += exp2f(ap.em2 * l);
    }
  }
}

// P = [x]_+^e (Eq. 2) and U = P^{2−α} = [x]_+^{e−1} (P:L377, 0 off the support).
template <int E>
__device__ __forceinline__ void p_and_u(float x, const AlphaParams& ap, float& p, float& u) {
  if (E == 1) {
    p = fmaxf(x, 0.f);
    u = (x > 0.f) ? 1.f : 0.f;
  } else if (E == 2) {
    u = fmaxf(x, 0.f);
    p = u * u;
  } else if (E == 4) {
    float xp = fmaxf(x, 0.f);
    float x2 = xp * xp;
    u = x2 * xp;
    p = x2 * x2;
  } else {
    if (x > 0.f) {
      float l = __log2f(x);
      p = exp2f(ap.e * l);
      u = exp2f(ap.em1 * l);
    } else {
      p = 0.f;
      u = 0.f;
    }
  }
}

// ---- packed f32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2): two lanes of work per issue slot
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmul.rn.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tadd.rn.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__device__ __forceinline__ float2 fabs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
// two floats → bf16x2 (RN) with relu: one F2FP.RELU; lo lands in the low half
__device__ __forceinline__ uint32_t pack_relu_bf16(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// P̂ = bf16([x]_+^e) and Û = bf16([x]_+^{e−1}) for e ∈ {2, 4} straight from x, without a separate relu:
// sign-carrying powers (x·|x|, …: the |·| is a free FMUL2 operand modifier) and relu inside the pack.
// Bitwise the same values as p_and_u + pack (x·|x| = x·x for x > 0; x <= 0 packs to ±0).
template <int E>
__device__ __forceinline__ void pu_packed(float2 x, uint32_t& pb, uint32_t& ub) {
  static_assert(E == 2 || E == 4, "integer exponents 2, 4");
  const float2 a = fmul2(x, fabs2(x));                 // x|x|  (= x² for x > 0)
  if constexpr (E == 2) {
    pb = pack_relu_bf16(a.x, a.y);
    ub = pack_relu_bf16(x.x, x.y);
  } else {
    const float2 b = fmul2(a, fabs2(x));               // x³ with x's sign
    const float2 c = fmul2(a, fabs2(a));               // x⁴ with x's sign
    pb = pack_relu_bf16(c.x, c.y);
    ub = pack_relu_bf16(b.x, b.y);
  }
}

// Generic α: U = x^{e−1} = 2^{(e−1)·log2 x} and P = U·x for a pair of x with two
// MUFU ops per element (lg2.approx.ftz, ex2.approx.ftz) and three other instructions, instead of an
// accurate exp2f per power (the tensor-core kernels are issue-bound there, so the instruction count is
// what matters: an FMA-pipe polynomial exp2 measured slower).  Relative error of U, P ≈ 2^-21·max(1,
// (e−1)·|log2 x|) — far below the bf16 rounding (2^-9) they get as MMA operands.  x <= 0 (or −∞ for
// masked keys) gives exactly 0; ex2.approx.ftz flushes an underflowing U to 0.
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void pu_generic2(float2 x, float em1, float2& p, float2& u) {
  const float2 y = fmul2(make_float2(lg2_approx(x.x), lg2_approx(x.y)), make_float2(em1, em1));
  u = make_float2(x.x > 0.f ? ex2_approx(y.x) : 0.f, x.y > 0.f ? ex2_approx(y.y) : 0.f);
  p = fmul2(u, make_float2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f)));
}

// P and U for a pair of x values (same semantics as p_and_u), FMA-pipe friendly for E = 1, 2 and the
// generic α path (E = 0).
template <int E>
__device__ __forceinline__ void p_and_u2(float2 x, const AlphaParams& ap, float2& p, float2& u) {
  if (E == 0) {
    pu_generic2(x, ap.em1, p, u);
  } else if (E == 2) {
    u = make_float2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f));
    p = fmul2(u, u);
  } else if (E == 1) {
    p = make_float2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f));
    u = make_float2(x.x > 0.f ? 1.f : 0.f, x.y > 0.f ? 1.f : 0.f);
  } else {
    p_and_u<E>(x.x, ap, p.x, u.x);
    p_and_u<E>(x.y, ap, p.y, u.y);
  }
}

// Alg. 1 state of one row.
struct RowState {
  float lo, hi, tau;
};

// Alg. 1 lines 4-6: τ_lo = m − 1, τ_hi = m − n^{1−α}, τ = midpoint.
__device__ __forceinline__ RowState bracket_init(float zmax, float n_visible, float alpha) {
  RowState s;
  s.lo = zmax - 1.0f;
  s.hi = zmax - exp2f((1.0f - alpha) * __log2f(n_visible));
  s.tau = 0.5f * (s.lo + s.hi);
  return s;
}

// One Alg. 1 iteration given the accumulated sums at the current τ (lines 8-14):
// bracket update (Eq. 4, tie f = 0 → τ_lo = τ), Halley candidate (Eq. 5), accept iff it lies in
// the updated bracket (inclusive) and is finite, else midpoint.
// Finite-precision reading (DESIGN.md r5): a candidate within a few fp32 ulps outside the bracket is
// accepted and clamped to it.  In exact arithmetic this is Alg. 1 itself; it matters when τ* sits on
// the bracket end (e.g. a single-element support gives τ* = τ_lo = m − 1, which the Newton/Halley
// step reaches exactly in real arithmetic but may overshoot by an ulp in fp32, which would otherwise
// demote the row to linear bisection for every remaining iteration).
__device__ __forceinline__ void alg1_update(RowState& s, float a0, float a1, float a2, const AlphaParams& ap) {
  float f = a0 - 1.0f;         // Eq. 3
  float f1 = ap.c1 * a1;       // Eq. 6
  float f2 = ap.c2 * a2;       // Eq. 7
  if (f < 0.f) s.hi = s.tau; else s.lo = s.tau;
  float den = 2.0f * f1 * f1 - f * f2;
  float th = s.tau - 2.0f * f * f1 / den;
  const float slack = 8.0f * 1.1920929e-7f * fmaxf(fabsf(s.lo), fabsf(s.hi));   // 8 ulp
  bool ok = (den != 0.f) && isfinite(th) && th >= s.lo - slack && th <= s.hi + slack;
  s.tau = ok ? fminf(fmaxf(th, s.lo), s.hi) : 0.5f * (s.lo + s.hi);
}

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Geometry of one call, passed by value to every kernel.
struct Geom {
  int B, H, N, d;
  long long sb, sh, sn;   // element strides of [B,H,N,d] tensors
  int Tr, Tc;             // ⌈N/B_r⌉, ⌈N/B_c⌉
  int causal;
  __host__ __device__ long long head_off(int bh) const {
    int b = bh / H, h = bh - (bh / H) * H;
    return (long long)b * sb + (long long)h * sh;
  }
  // number of key blocks visible to query block i (causal: blocks j with j*Bc <= last row of i)
  __host__ __device__ int visible_kblocks(int i) const {
    if (!causal) return Tc;
    int last_row = min(N, (i + 1) * kBr) - 1;
    return last_row / kBc + 1;
  }
};

}  // namespace entmax
