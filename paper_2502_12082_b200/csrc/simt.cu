// simt.cu — launchers of the SIMT fp32-arithmetic kernels and of the small shared kernels.
#include "entmax_attn.h"
#include "runtime.h"
#include "simt_kernels.cuh"

namespace entmax {
namespace {

template <typename T, int D, int E>
int fwd_impl(const void* q, const void* k, const void* v, const Geom& g, const AlphaParams& ap, int n_iter, void* o,
             void* o2, float* tau, uint8_t* mask, int32_t* row_cnt, int32_t* row_idx, cudaStream_t st) {
  dim3 grid(g.Tr, g.B * g.H);
  {
    ProfScope ps("simt_tau", st);
    simt::tau_kernel<T, D, E><<<grid, 128, 0, st>>>((const T*)q, (const T*)k, g, ap, n_iter, tau);
  }
  if (int rc = cuda_status("simt_tau")) return rc;
  {
    ProfScope ps("simt_out", st);
    simt::out_kernel<T, D, E><<<grid, 128, 0, st>>>((const T*)q, (const T*)k, (const T*)v, g, ap, tau, (T*)o,
                                                    (float*)o2, mask, row_cnt, row_idx);
  }
  return cuda_status("simt_out");
}

template <typename T, int D, int E>
int bwd_impl(const void* q, const void* k, const void* v, const void* dO, const Geom& g, const AlphaParams& ap,
             const float* tau, const float* delta, const int32_t* row_cnt, const int32_t* row_idx,
             const int32_t* col_cnt, const int32_t* col_idx, void* dq, void* dk, void* dv, cudaStream_t st) {
  {
    ProfScope ps("simt_dkdv", st);
    simt::dkdv_kernel<T, D, E><<<dim3(g.Tc, g.B * g.H), 128, 0, st>>>(
        (const T*)q, (const T*)k, (const T*)v, (const T*)dO, g, ap, tau, delta, col_cnt, col_idx, (T*)dk, (T*)dv);
  }
  if (int rc = cuda_status("simt_dkdv")) return rc;
  {
    ProfScope ps("simt_dq", st);
    simt::dq_kernel<T, D, E><<<dim3(g.Tr, g.B * g.H), 128, 0, st>>>(
        (const T*)q, (const T*)k, (const T*)v, (const T*)dO, g, ap, tau, delta, row_cnt, row_idx, (T*)dq);
  }
  return cuda_status("simt_dq");
}

// (dtype, d, ecode) → template instance
template <template <typename, int, int> class Op, typename... Args>
int dispatch(int dtype, int d, int ecode, Args&&... args) {
#define ENTMAX_CASE_E(T, D)                                                  \
  switch (ecode) {                                                           \
    case 1: return Op<T, D, 1>::run(args...);                                \
    case 2: return Op<T, D, 2>::run(args...);                                \
    case 4: return Op<T, D, 4>::run(args...);                                \
    default: return Op<T, D, 0>::run(args...);                               \
  }
#define ENTMAX_CASE_D(T)                                                     \
  switch (d) {                                                               \
    case 16: ENTMAX_CASE_E(T, 16)                                            \
    case 32: ENTMAX_CASE_E(T, 32)                                            \
    case 64: ENTMAX_CASE_E(T, 64)                                            \
    case 128: ENTMAX_CASE_E(T, 128)                                          \
    default: return fail(ENTMAX_ERR_UNSUPPORTED, "head dim %d not supported by the SIMT kernels", d); \
  }
  if (dtype == ENTMAX_FP32) {
    ENTMAX_CASE_D(float)
  } else {
    ENTMAX_CASE_D(__nv_bfloat16)
  }
#undef ENTMAX_CASE_D
#undef ENTMAX_CASE_E
}

template <typename T, int D, int E>
struct FwdOp {
  template <typename... A>
  static int run(A&&... a) { return fwd_impl<T, D, E>(a...); }
};
template <typename T, int D, int E>
struct BwdOp {
  template <typename... A>
  static int run(A&&... a) { return bwd_impl<T, D, E>(a...); }
};

}  // namespace

int simt_fwd_launch(int dtype, int d, int ecode, const void* q, const void* k, const void* v, const Geom& g,
                    const AlphaParams& ap, int n_iter, void* o, void* o2, float* tau, uint8_t* mask,
                    int32_t* row_cnt, int32_t* row_idx, cudaStream_t st) {
  return dispatch<FwdOp>(dtype, d, ecode, q, k, v, g, ap, n_iter, o, o2, tau, mask, row_cnt, row_idx, st);
}

int simt_bwd_launch(int dtype, int d, int ecode, const void* q, const void* k, const void* v, const void* dO,
                    const Geom& g, const AlphaParams& ap, const float* tau, const float* delta,
                    const int32_t* row_cnt, const int32_t* row_idx, const int32_t* col_cnt, const int32_t* col_idx,
                    void* dq, void* dk, void* dv, cudaStream_t st) {
  return dispatch<BwdOp>(dtype, d, ecode, q, k, v, dO, g, ap, tau, delta, row_cnt, row_idx, col_cnt, col_idx, dq,
                         dk, dv, st);
}

template <typename T>
static void delta_go(const T* dO, const float* o2, const float* tau, const Geom& g, float* delta, float* td,
                     cudaStream_t st) {
  const long long rows = (long long)g.B * g.H * g.Tr * kBr;   // padded rows (td staging)
  const int tpr = g.d / 8;
  const unsigned blocks = (unsigned)((rows * tpr + 255) / 256);
  switch (tpr) {
    case 2: launch_pdl(delta_kernel<T, 2>, dim3(blocks), dim3(256), 0, st, dO, o2, tau, g, delta, td); break;
    case 4: launch_pdl(delta_kernel<T, 4>, dim3(blocks), dim3(256), 0, st, dO, o2, tau, g, delta, td); break;
    case 8: launch_pdl(delta_kernel<T, 8>, dim3(blocks), dim3(256), 0, st, dO, o2, tau, g, delta, td); break;
    default: launch_pdl(delta_kernel<T, 16>, dim3(blocks), dim3(256), 0, st, dO, o2, tau, g, delta, td); break;
  }
}

int delta_launch(int dtype, const void* dO, const void* o2, const float* tau, const Geom& g, float* delta, float* td,
                 cudaStream_t st) {
  if (g.d != 16 && g.d != 32 && g.d != 64 && g.d != 128) return fail(ENTMAX_ERR_UNSUPPORTED, "delta: d = %d not supported", g.d);
  {
    ProfScope ps("delta", st);
    if (dtype == ENTMAX_FP32)
      delta_go<float>(static_cast<const float*>(dO), static_cast<const float*>(o2), tau, g, delta, td, st);
    else
      delta_go<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(dO), static_cast<const float*>(o2), tau, g, delta, td,
                              st);
  }
  return cuda_status("delta");
}

int col_lists_launch(const uint8_t* mask, const Geom& g, int32_t* col_cnt, int32_t* col_idx, cudaStream_t st) {
  const long long n = (long long)g.B * g.H * g.Tc;
  {
    ProfScope ps("col_lists", st);
    launch_pdl(col_lists_kernel, dim3((unsigned)((n * 32 + 255) / 256)), dim3(256), 0, st, mask, g.B * g.H, g.Tr,
               g.Tc, col_cnt, col_idx);   // one warp per (head, key block)
  }
  return cuda_status("col_lists");
}

}  // namespace entmax

extern "C" int entmax_attn_pack_mask(const uint8_t* mask, int64_t rows, int32_t Tc, uint32_t* out, void* stream) {
  using namespace entmax;
  if (!mask || !out) return fail(ENTMAX_ERR_INVALID_ARG, "NULL pointer");
  if (rows < 1 || Tc < 1) return fail(ENTMAX_ERR_INVALID_ARG, "rows and Tc must be >= 1");
  const int words = (Tc + 31) / 32;
  const long long n = rows * words;
  pack_mask_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(mask, rows, Tc, words, out);
  return cuda_status("pack_mask");
}
