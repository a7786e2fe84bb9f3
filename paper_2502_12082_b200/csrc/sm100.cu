// sm100.cu — host launchers of the tcgen05 / TMEM / TMA kernels (sm100_kernels.cuh).
#include "entmax_attn.h"
#include "runtime.h"
#include "sm100_kernels.cuh"
#include "sm100_tau.cuh"
#include "sm100_fb.cuh"
#include "sm100_fb2.cuh"
#include "tmap.h"

namespace entmax {
namespace sm100 {
namespace {

template <int D>
constexpr size_t out_smem(int Tc) {
  return 1024 + Cfg<D>::TILE + ((D == 64) ? 6 : 2) * 2 * Cfg<D>::TILE + 2 * kFbMath * 4 + (size_t)Tc;
}
template <int D>
constexpr size_t dkdv_smem() {
  return 1024 + 2 * Cfg<D>::TILE + ((D == 64) ? 5 : 2) * (2 * Cfg<D>::TILE + 1024);
}
template <int D>
constexpr size_t dq_smem() {
  return 1024 + 2 * Cfg<D>::TILE + ((D == 64) ? 5 : 2) * 2 * Cfg<D>::TILE + kOnesBytes;
}

#ifndef ENTMAX_OUT_MW
#define ENTMAX_OUT_MW 8     // math warps of the (1-SM) output kernel (16 measured 1.03 -> 1.05 ms at config 2)
#endif
constexpr int kOutMW = ENTMAX_OUT_MW;
#ifndef ENTMAX_DQ_MW
#define ENTMAX_DQ_MW 8      // math warps of the dQ kernel (16 measured slower: 1.075 -> 1.133 ms at config 2)
#endif
#ifndef ENTMAX_DKDV_MW
#define ENTMAX_DKDV_MW 16   // math warps of the dK/dV kernel (8: 1.64 ms, 16: 1.43 ms at config 2)
#endif

constexpr size_t kMaxSmem = 232448;  // 227 KB opt-in per block on sm_100

template <typename K>
int set_smem(K kernel, size_t bytes) {
  if (bytes > kMaxSmem) return fail(ENTMAX_ERR_UNSUPPORTED, "kernel needs %zu B of shared memory", bytes);
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(ENTMAX_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  return ENTMAX_OK;
}

int tmaps(const Geom& g, std::initializer_list<std::pair<CUtensorMap*, const void*>> maps) {
  for (auto& m : maps)
    if (!make_tmap_bhnd(m.first, m.second, g.B, g.H, g.N, g.d, g.sb, g.sh, g.sn))
      return fail(ENTMAX_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (alignment/strides?)");
  return ENTMAX_OK;
}

template <int D, int E, bool CU>
int fwd_t(const void* q, const void* k, const void* v, const Geom& g, const AlphaParams& ap, int n_iter, void* o,
          void* o2, float* tau, uint8_t* mask, int32_t* row_cnt, int32_t* row_idx, int32_t* cand_cnt,
          int32_t* cand_idx, cudaStream_t st) {
  CUtensorMap tq, tk, tv, tk64;
  if (int rc = tmaps(g, {{&tq, q}, {&tk, k}, {&tv, v}})) return rc;
  if (!make_tmap_bhnd(&tk64, k, g.B, g.H, g.N, g.d, g.sb, g.sh, g.sn, 64))
    return fail(ENTMAX_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (64-row K boxes)");
  const dim3 grid(g.Tr, g.B * g.H);
  {
    const size_t sm = TauSmem<D>::bytes(g.Tc);
    if (int rc = set_smem(tau_kernel<D, E>, sm)) return rc;
    ProfScope ps("tau_sm100", st);
    if (cudaError_t e = launch_pdl(tau_kernel<D, E>, dim3(g.Tr, g.B * g.H), dim3(kTauThreads), sm, st, tq,
                                   tk, g, ap, n_iter, tau, cand_cnt, cand_idx))
      return fail(ENTMAX_ERR_CUDA, "tau_sm100 launch: %s", cudaGetErrorString(e));
  }
  if (int rc = cuda_status("tau_sm100")) return rc;
#ifndef ENTMAX_OUT1   // diagnostics: the 1-SM output kernel at d = 128 too
  // d = 128: output pass on CTA pairs (2-SM MMAs, sm100_fb2.cuh), measured 16 % faster at config 5
  // (N = 32768 causal: 5.66 → 4.76 ms).  d = 64 keeps the 1-SM kernel: there a tile's MMAs take half as
  // long and the pair's cross-CTA P handshake is no longer hidden (1.03 → 1.59 ms at config 2).
  if constexpr (D == 128) {
    // V halves as MN-major SW128 boxes (SW64 [128 × 32] boxes would serve d = 64)
    CUtensorMap tvh;
    const bool ok = D == 64 ? make_tmap_bhnd_sw64(&tvh, v, g.B, g.H, g.N, g.d, g.sb, g.sh, g.sn)
                            : make_tmap_bhnd(&tvh, v, g.B, g.H, g.N, g.d, g.sb, g.sh, g.sn);
    if (!ok) return fail(ENTMAX_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (V halves)");
    const size_t sm2 = Out2Cfg<D>::smem(g.Tc);
    const dim3 grid2((g.Tr + 1) & ~1, g.B * g.H);
    ProfScope ps("out_sm100", st);
    cudaError_t e;
    if (o2 != nullptr) {
      if (int rc = set_smem(out2_kernel<D, E, true, CU>, sm2)) return rc;
      e = launch_pdl(out2_kernel<D, E, true, CU>, grid2, dim3(kFbThreads), sm2, st, tq, tk64, tvh, g, ap, tau, cand_cnt,
                     cand_idx, (__nv_bfloat16*)o, (float*)o2, mask, row_cnt, row_idx);
    } else {
      if (int rc = set_smem(out2_kernel<D, E, false, CU>, sm2)) return rc;
      e = launch_pdl(out2_kernel<D, E, false, CU>, grid2, dim3(kFbThreads), sm2, st, tq, tk64, tvh, g, ap, tau, cand_cnt,
                     cand_idx, (__nv_bfloat16*)o, (float*)nullptr, mask, row_cnt, row_idx);
    }
    if (e != cudaSuccess) return fail(ENTMAX_ERR_CUDA, "out_sm100 launch: %s", cudaGetErrorString(e));
    return cuda_status("out_sm100");
  }
#endif
  const size_t sm = out_smem<D>(g.Tc);
  if (o2 != nullptr) {
    if (int rc = set_smem(out_kernel<D, E, true, CU, kOutMW>, sm)) return rc;
    ProfScope ps("out_sm100", st);
    if (cudaError_t e = launch_pdl(out_kernel<D, E, true, CU, kOutMW>, grid, dim3(out_threads<kOutMW>()), sm, st, tq, tk, tv, g, ap, tau,
                                   cand_cnt, cand_idx, (__nv_bfloat16*)o, (float*)o2, mask, row_cnt, row_idx))
      return fail(ENTMAX_ERR_CUDA, "out_sm100 launch: %s", cudaGetErrorString(e));
  } else {
    if (int rc = set_smem(out_kernel<D, E, false, CU, kOutMW>, sm)) return rc;
    ProfScope ps("out_sm100", st);
    if (cudaError_t e = launch_pdl(out_kernel<D, E, false, CU, kOutMW>, grid, dim3(out_threads<kOutMW>()), sm, st, tq, tk, tv, g, ap, tau,
                                   cand_cnt, cand_idx, (__nv_bfloat16*)o, (float*)nullptr, mask, row_cnt, row_idx))
      return fail(ENTMAX_ERR_CUDA, "out_sm100 launch: %s", cudaGetErrorString(e));
  }
  return cuda_status("out_sm100");
}

template <int D, int E, bool CU>
int bwd_t(const void* q, const void* k, const void* v, const void* dO, const Geom& g, const AlphaParams& ap,
          const float* tau, const float* delta, const int32_t* row_cnt, const int32_t* row_idx,
          const int32_t* col_cnt, const int32_t* col_idx, const float* td, float* kbar, void* dq, void* dk, void* dv,
          cudaStream_t st) {
  CUtensorMap tq, tk, tv, tdo;
  if (int rc = tmaps(g, {{&tq, q}, {&tk, k}, {&tv, v}, {&tdo, dO}})) return rc;
  {
    const size_t sm = dkdv_smem<D>();
    constexpr int MW = ENTMAX_DKDV_MW;
    if (int rc = set_smem(dkdv_kernel<D, E, CU, MW>, sm)) return rc;
    ProfScope ps("dkdv_sm100", st);
    if (cudaError_t e = launch_pdl(dkdv_kernel<D, E, CU, MW>, dim3(g.Tc, g.B * g.H), dim3(dkdv_threads<MW>()), sm, st, tq, tk, tv, tdo,
                                   g, ap, td, col_cnt, col_idx, kbar, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv))
      return fail(ENTMAX_ERR_CUDA, "dkdv_sm100 launch: %s", cudaGetErrorString(e));
  }
  if (int rc = cuda_status("dkdv_sm100")) return rc;
  {
    const size_t sm = dq_smem<D>();
    constexpr int MW = ENTMAX_DQ_MW;
    if (int rc = set_smem(dq_kernel<D, E, CU, MW>, sm)) return rc;
    ProfScope ps("dq_sm100", st);
    if (cudaError_t e = launch_pdl(dq_kernel<D, E, CU, MW>, dim3(g.Tr, g.B * g.H), dim3(dq_threads<MW>()), sm, st, tq, tk, tv, tdo, g,
                                   ap, tau, delta, row_cnt, row_idx, kbar, (__nv_bfloat16*)dq))
      return fail(ENTMAX_ERR_CUDA, "dq_sm100 launch: %s", cudaGetErrorString(e));
  }
  return cuda_status("dq_sm100");
}

template <template <int, int> class Op, typename... A>
int dispatch(int d, int ecode, A&&... a) {
#define ENTMAX_E(DD)                                   \
  switch (ecode) {                                     \
    case 1: return Op<DD, 1>::run(a...);               \
    case 2: return Op<DD, 2>::run(a...);               \
    case 4: return Op<DD, 4>::run(a...);               \
    default: return Op<DD, 0>::run(a...);              \
  }
  if (d == 64) ENTMAX_E(64)
  if (d == 128) ENTMAX_E(128)
#undef ENTMAX_E
  return fail(ENTMAX_ERR_UNSUPPORTED, "tcgen05 path supports d in {64, 128} (got %d)", d);
}

// (the first argument after the inputs is the Geom: short rows select the consistent-Û kernels, r9)
template <int D, int E>
struct FwdOp {
  template <typename Q, typename K, typename V, typename... A>
  static int run(Q q, K k, V v, const Geom& g, A&&... a) {
    return g.N <= kConsistentUMaxN ? fwd_t<D, E, true>(q, k, v, g, a...) : fwd_t<D, E, false>(q, k, v, g, a...);
  }
};
template <int D, int E>
struct BwdOp {
  template <typename Q, typename K, typename V, typename O, typename... A>
  static int run(Q q, K k, V v, O dO, const Geom& g, A&&... a) {
    return g.N <= kConsistentUMaxN ? bwd_t<D, E, true>(q, k, v, dO, g, a...) : bwd_t<D, E, false>(q, k, v, dO, g, a...);
  }
};

}  // namespace

bool available() {
  static const bool ok = [] {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0 && tmap_encoder() != nullptr;
  }();
  return ok;
}

int fwd(const void* q, const void* k, const void* v, const Geom& g, const AlphaParams& ap, int ecode, int n_iter,
        void* o, void* o2, float* tau, uint8_t* mask, int32_t* row_cnt, int32_t* row_idx, int32_t* cand_cnt,
        int32_t* cand_idx, cudaStream_t st) {
  return dispatch<FwdOp>(g.d, ecode, q, k, v, g, ap, n_iter, o, o2, tau, mask, row_cnt, row_idx, cand_cnt, cand_idx,
                         st);
}

int bwd(const void* q, const void* k, const void* v, const void* dO, const Geom& g, const AlphaParams& ap, int ecode,
        const float* tau, const float* delta, const int32_t* row_cnt, const int32_t* row_idx, const int32_t* col_cnt,
        const int32_t* col_idx, const float* td, float* kbar, void* dq, void* dk, void* dv, cudaStream_t st) {
  return dispatch<BwdOp>(g.d, ecode, q, k, v, dO, g, ap, tau, delta, row_cnt, row_idx, col_cnt, col_idx, td, kbar, dq,
                         dk, dv, st);
}

}  // namespace sm100
}  // namespace entmax
