// trace_api.cu — exports the trace buffer of the diagnostics build (-DENTMAX_TRACE).
#include <cuda_runtime.h>
namespace entmax {
__device__ unsigned long long g_trace[8192];
__device__ int g_trace_bx;
__device__ int g_trace_kid;
}
extern "C" int entmax_trace_reset(int bx) {
  unsigned long long z[8192] = {};
  cudaMemcpyToSymbol(entmax::g_trace, z, sizeof(z));
  return cudaMemcpyToSymbol(entmax::g_trace_bx, &bx, sizeof(int)) == cudaSuccess ? 0 : 1;
}
extern "C" int entmax_trace_kernel(int kid) {
  return cudaMemcpyToSymbol(entmax::g_trace_kid, &kid, sizeof(int)) == cudaSuccess ? 0 : 1;
}
extern "C" int entmax_trace_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, entmax::g_trace, sizeof(unsigned long long) * 8192) == cudaSuccess ? 0 : 1;
}
