// entmax_attn.cu — C ABI (include/entmax_attn.h): validation, workspace carve-up, dispatch
// to the tcgen05 (sm_100a) or SIMT kernels, optional per-kernel event timing.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "entmax_attn.h"
#include "common.cuh"
#include "runtime.h"

using namespace entmax;

// ---------------------------------------------------------------------------------------
// error reporting
// ---------------------------------------------------------------------------------------
namespace {
thread_local std::string g_last_error;

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_pending;
std::vector<cudaEvent_t> g_event_pool;
struct ProfAgg {
  const char* name;
  int launches;
  double ms;
};
std::vector<ProfAgg> g_prof_agg;

cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct FwdWs {
  size_t cand_cnt, cand_idx, total;
};
struct BwdWs {
  size_t delta, col_cnt, col_idx, kbar, td, total;
};

FwdWs fwd_ws_layout(const entmax_shape_t& s) {
  const size_t BH = (size_t)s.B * s.H;
  const size_t Tr = (s.N + kBr - 1) / kBr, Tc = (s.N + kBc - 1) / kBc;
  FwdWs w;
  w.cand_cnt = 0;
  w.cand_idx = align256(w.cand_cnt + BH * Tr * sizeof(int32_t));
  w.total = align256(w.cand_idx + BH * Tr * Tc * sizeof(int32_t));
  return w;
}

BwdWs bwd_ws_layout(const entmax_shape_t& s) {
  const size_t BH = (size_t)s.B * s.H;
  const size_t Tr = (s.N + kBr - 1) / kBr, Tc = (s.N + kBc - 1) / kBc;
  BwdWs w;
  w.delta = 0;
  w.col_cnt = align256(BH * s.N * sizeof(float));
  w.col_idx = align256(w.col_cnt + BH * Tc * sizeof(int32_t));
  // K̄_j: per-key-block mean key (fp32), written by the dK/dV kernel for dQ's leak correction (r12)
  w.kbar = align256(w.col_idx + BH * Tc * Tr * sizeof(int32_t));
  // td: per query block {τ[128] | δ[128]} (+∞ / 0 past N), the dK/dV producer's bulk-copy source
  w.td = align256(w.kbar + BH * Tc * (size_t)s.d * sizeof(float));
  w.total = align256(w.td + BH * Tr * 2 * kBr * sizeof(float));
  return w;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_shape(const entmax_shape_t* s, int dtype) {
  if (!s) return fail(ENTMAX_ERR_INVALID_ARG, "shape pointer is NULL");
  if (s->B < 1 || s->H < 1 || s->N < 1 || s->d < 1)
    return fail(ENTMAX_ERR_INVALID_ARG, "B, H, N, d must be >= 1 (got %d %d %d %d)", s->B, s->H, s->N, s->d);
  if (dtype != ENTMAX_BF16 && dtype != ENTMAX_FP32) return fail(ENTMAX_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (s->sn < s->d || s->sh < (int64_t)s->N * s->sn || s->sb < (int64_t)s->H * s->sh)
    return fail(ENTMAX_ERR_INVALID_ARG, "strides (sb=%lld sh=%lld sn=%lld) overlap rows/heads",
                (long long)s->sb, (long long)s->sh, (long long)s->sn);
  const int esz = dtype == ENTMAX_BF16 ? 2 : 4;
  if ((s->sn * esz) % 16 || (s->sh * esz) % 16 || (s->sb * esz) % 16 || (s->d * esz) % 16)
    return fail(ENTMAX_ERR_INVALID_ARG, "strides and d must be multiples of 16 bytes");
  if ((int64_t)s->N * 1 > (1 << 24)) return fail(ENTMAX_ERR_UNSUPPORTED, "N > 2^24 not supported");
  if ((int64_t)s->B * s->H > 65535)   // heads are the grid's y dimension
    return fail(ENTMAX_ERR_UNSUPPORTED, "B*H = %lld > 65535 heads per call: split the batch",
                (long long)s->B * s->H);
  return ENTMAX_OK;
}

int check_alpha(float alpha) {
  if (!(alpha >= 1.001f)) return fail(ENTMAX_ERR_INVALID_ARG, "alpha must be >= 1 + 1e-3 (got %g)", alpha);
  if (alpha > 2.0f) return fail(ENTMAX_ERR_UNSUPPORTED, "alpha > 2 not supported (got %g)", alpha);
  return ENTMAX_OK;
}

int impl_for(const entmax_shape_t& s, int dtype) {
  static const bool force_simt = [] {
    const char* e = getenv("ENTMAX_ATTN_FORCE_SIMT");
    return e && e[0] == '1';
  }();
  if (dtype == ENTMAX_BF16 && (s.d == 64 || s.d == 128) && !force_simt && sm100::available()) return 1;
  if (s.d == 16 || s.d == 32 || s.d == 64 || s.d == 128) return 0;
  return -1;
}

Geom make_geom(const entmax_shape_t& s, int causal) {
  Geom g;
  g.B = s.B;
  g.H = s.H;
  g.N = s.N;
  g.d = s.d;
  g.sb = s.sb;
  g.sh = s.sh;
  g.sn = s.sn;
  g.Tr = (s.N + kBr - 1) / kBr;
  g.Tc = (s.N + kBc - 1) / kBc;
  g.causal = causal ? 1 : 0;
  return g;
}

}  // namespace

namespace entmax {

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ENTMAX_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return ENTMAX_OK;
}

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  on = g_prof_on;
  if (on) {
    a = get_event();
    b = get_event();
    cudaEventRecord(a, st);
  }
}

ProfScope::~ProfScope() {
  if (!on) return;
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_pending.push_back({name, a, b});
}

}  // namespace entmax

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

const char* entmax_attn_status_string(int status) {
  switch (status) {
    case ENTMAX_OK: return "ok";
    case ENTMAX_ERR_INVALID_ARG: return "invalid argument";
    case ENTMAX_ERR_UNSUPPORTED: return "unsupported configuration";
    case ENTMAX_ERR_WORKSPACE: return "workspace too small";
    case ENTMAX_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char* entmax_attn_last_error(void) { return g_last_error.c_str(); }

int entmax_attn_block_size(int32_t d, int dtype, int32_t* Br, int32_t* Bc) {
  if (dtype != ENTMAX_BF16 && dtype != ENTMAX_FP32) return fail(ENTMAX_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (d != 16 && d != 32 && d != 64 && d != 128) return fail(ENTMAX_ERR_UNSUPPORTED, "head dim %d not supported", d);
  if (Br) *Br = kBr;
  if (Bc) *Bc = kBc;
  return ENTMAX_OK;
}

size_t entmax_attn_fwd_workspace_bytes(const entmax_shape_t* shp, int dtype, int causal) {
  (void)dtype;
  (void)causal;
  if (!shp || shp->B < 1 || shp->H < 1 || shp->N < 1) return 0;
  return fwd_ws_layout(*shp).total;
}

size_t entmax_attn_bwd_workspace_bytes(const entmax_shape_t* shp, int dtype, int causal) {
  (void)dtype;
  (void)causal;
  if (!shp || shp->B < 1 || shp->H < 1 || shp->N < 1) return 0;
  return bwd_ws_layout(*shp).total;
}

int entmax_attn_impl_for(const entmax_shape_t* shp, int dtype) {
  if (!shp) return -1;
  return impl_for(*shp, dtype);
}

int entmax_attn_fwd(const void* q, const void* k, const void* v, const entmax_shape_t* shp, int dtype, float alpha,
                    int causal, int n_iter, float scale, void* o, void* o2, float* tau, uint8_t* mask,
                    int32_t* row_cnt, int32_t* row_idx, void* workspace, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (int rc = check_shape(shp, dtype)) return rc;
  if (int rc = check_alpha(alpha)) return rc;
  if (n_iter < 1) return fail(ENTMAX_ERR_INVALID_ARG, "n_iter must be >= 1 (got %d)", n_iter);
  if (!q || !k || !v || !o || !tau) return fail(ENTMAX_ERR_INVALID_ARG, "NULL tensor pointer");
  // mask, row_cnt, row_idx: all set (block-sparse mode) or all NULL (unmasked mode, NEXT-2)
  if ((mask == nullptr) != (row_cnt == nullptr) || (mask == nullptr) != (row_idx == nullptr))
    return fail(ENTMAX_ERR_INVALID_ARG, "mask, row_cnt and row_idx must be all set or all NULL (unmasked mode)");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || (o2 && !aligned16(o2)))
    return fail(ENTMAX_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const FwdWs wl = fwd_ws_layout(*shp);
  if (ws_bytes < wl.total || (wl.total && !workspace))
    return fail(ENTMAX_ERR_WORKSPACE, "forward workspace needs %zu bytes (got %zu)", wl.total, ws_bytes);
  const int impl = impl_for(*shp, dtype);
  if (impl < 0) return fail(ENTMAX_ERR_UNSUPPORTED, "head dim %d / dtype %d not supported", shp->d, dtype);
  if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)shp->d);
  const Geom g = make_geom(*shp, causal);
  const AlphaParams ap = make_alpha_params(alpha, scale);
  const int ecode = exponent_code(alpha);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  if (impl == 1) {
    return sm100::fwd(q, k, v, g, ap, ecode, n_iter, o, o2, tau, mask, row_cnt, row_idx,
                      (int32_t*)(ws + wl.cand_cnt), (int32_t*)(ws + wl.cand_idx), st);
  }
  return simt_fwd_launch(dtype, shp->d, ecode, q, k, v, g, ap, n_iter, o, o2, tau, mask, row_cnt, row_idx, st);
}

int entmax_attn_bwd(const void* q, const void* k, const void* v, const void* o2, const void* d_o, const float* tau,
                    const uint8_t* mask, const int32_t* row_cnt, const int32_t* row_idx, const entmax_shape_t* shp,
                    int dtype, float alpha, int causal, float scale, void* dq, void* dk, void* dv, void* workspace,
                    size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (int rc = check_shape(shp, dtype)) return rc;
  if (int rc = check_alpha(alpha)) return rc;
  if (!q || !k || !v || !o2 || !d_o || !tau || !dq || !dk || !dv) return fail(ENTMAX_ERR_INVALID_ARG, "NULL tensor pointer");
  if ((mask == nullptr) != (row_cnt == nullptr) || (mask == nullptr) != (row_idx == nullptr))
    return fail(ENTMAX_ERR_INVALID_ARG, "mask, row_cnt and row_idx must be all set or all NULL (unmasked mode)");
  const bool unmasked = mask == nullptr;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o2) || !aligned16(d_o) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv))
    return fail(ENTMAX_ERR_INVALID_ARG, "tensor pointers must be 16-byte aligned");
  const BwdWs wl = bwd_ws_layout(*shp);
  if (ws_bytes < wl.total || (wl.total && !workspace))
    return fail(ENTMAX_ERR_WORKSPACE, "backward workspace needs %zu bytes (got %zu)", wl.total, ws_bytes);
  const int impl = impl_for(*shp, dtype);
  if (impl < 0) return fail(ENTMAX_ERR_UNSUPPORTED, "head dim %d / dtype %d not supported", shp->d, dtype);
  if (!(scale > 0.f)) scale = 1.0f / sqrtf((float)shp->d);
  const Geom g = make_geom(*shp, causal);
  const AlphaParams ap = make_alpha_params(alpha, scale);
  const int ecode = exponent_code(alpha);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  float* delta = (float*)(ws + wl.delta);
  int32_t* col_cnt = unmasked ? nullptr : (int32_t*)(ws + wl.col_cnt);
  int32_t* col_idx = unmasked ? nullptr : (int32_t*)(ws + wl.col_idx);

  // δ and the 𝒦 tables — shared by both implementations; the unmasked
  // mode visits every visible block and needs no tables
  float* td = impl == 1 ? (float*)(ws + wl.td) : nullptr;
  if (int rc = delta_launch(dtype, d_o, o2, tau, g, delta, td, st)) return rc;
  if (!unmasked)
    if (int rc = col_lists_launch(mask, g, col_cnt, col_idx, st)) return rc;

  if (impl == 1) {
    return sm100::bwd(q, k, v, d_o, g, ap, ecode, tau, delta, row_cnt, row_idx, col_cnt, col_idx, td,
                      (float*)(ws + wl.kbar), dq, dk, dv, st);
  }
  return simt_bwd_launch(dtype, shp->d, ecode, q, k, v, d_o, g, ap, tau, delta, row_cnt, row_idx, col_cnt, col_idx, dq,
                         dk, dv, st);
}

void entmax_attn_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
}

void entmax_attn_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof_pending) {
    cudaEventSynchronize(r.b);
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_pending.clear();
  g_prof_agg.clear();
}

int entmax_attn_profile_collect(const char** names, int32_t* launches, double* total_ms, int cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& a : g_prof_agg)
      if (strcmp(a.name, r.name) == 0) {
        a.launches++;
        a.ms += ms;
        found = true;
        break;
      }
    if (!found) g_prof_agg.push_back({r.name, 1, (double)ms});
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_pending.clear();
  int n = 0;
  for (auto& a : g_prof_agg) {
    if (n >= cap) break;
    if (names) names[n] = a.name;
    if (launches) launches[n] = a.launches;
    if (total_ms) total_ms[n] = a.ms;
    ++n;
  }
  return n;
}

}  // extern "C"
