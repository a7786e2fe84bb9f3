// runtime.h — host-side helpers shared by the translation units of libentmax_attn.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace entmax {

// Record a failure detail for entmax_attn_last_error() and return `status`.
int fail(int status, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

// ENTMAX_ERR_CUDA with the launch error string if the last launch failed, else ENTMAX_OK.
int cuda_status(const char* where);

// CUDA-event bracket around one launch on `st` (active only when profiling is enabled).
struct ProfScope {
  const char* name;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  bool on = false;
  ProfScope(const char* n, cudaStream_t s);
  ~ProfScope();
};

// Launch with programmatic stream serialization (PDL): the kernel may start while the previous
// kernel of the stream drains; every kernel so launched calls griddepcontrol.wait before it touches
// global data (sm100_ptx.cuh griddep_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// SIMT path (simt.cu)
int simt_fwd_launch(int dtype, int d, int ecode, const void* q, const void* k, const void* v, const Geom& g,
                    const AlphaParams& ap, int n_iter, void* o, void* o2, float* tau, uint8_t* mask,
                    int32_t* row_cnt, int32_t* row_idx, cudaStream_t st);
int simt_bwd_launch(int dtype, int d, int ecode, const void* q, const void* k, const void* v, const void* dO,
                    const Geom& g, const AlphaParams& ap, const float* tau, const float* delta,
                    const int32_t* row_cnt, const int32_t* row_idx, const int32_t* col_cnt, const int32_t* col_idx,
                    void* dq, void* dk, void* dv, cudaStream_t st);
// shared small kernels (simt.cu)
int delta_launch(int dtype, const void* dO, const void* o2, const float* tau, const Geom& g, float* delta, float* td,
                 cudaStream_t st);
int col_lists_launch(const uint8_t* mask, const Geom& g, int32_t* col_cnt, int32_t* col_idx, cudaStream_t st);

// tcgen05 path (sm100.cu)
namespace sm100 {
bool available();
int fwd(const void* q, const void* k, const void* v, const Geom& g, const AlphaParams& ap, int ecode, int n_iter,
        void* o, void* o2, float* tau, uint8_t* mask, int32_t* row_cnt, int32_t* row_idx, int32_t* cand_cnt,
        int32_t* cand_idx, cudaStream_t st);
int bwd(const void* q, const void* k, const void* v, const void* dO, const Geom& g, const AlphaParams& ap, int ecode,
        const float* tau, const float* delta, const int32_t* row_cnt, const int32_t* row_idx, const int32_t* col_cnt,
        const int32_t* col_idx, const float* td, float* kbar, void* dq, void* dk, void* dv, cudaStream_t st);
}  // namespace sm100

}  // namespace entmax
