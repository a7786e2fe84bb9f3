// trace.cuh — optional pipeline tracing (diagnostics build only: -DENTMAX_TRACE).  Records
// clock64() timestamps of pipeline events of one CTA (blockIdx == (trace_bx, 0)) of one kernel
// (g_trace_kid: 0 τ, 1 output, 2 dK/dV, 3 dQ) into a device array that the diagnostics library
// exports; compiles to nothing in the product build.
#pragma once
#include <cstdint>

#ifdef ENTMAX_TRACE
namespace entmax {
extern __device__ unsigned long long g_trace[8192];
extern __device__ int g_trace_bx;
extern __device__ int g_trace_kid;
}
#define ENTMAX_TRACE_K(kid, slot)                                                                       \
  do {                                                                                                  \
    if (::entmax::g_trace_kid == (kid) && blockIdx.x == (unsigned)::entmax::g_trace_bx && blockIdx.y == 0 && \
        (slot) < 8192)                                                                                  \
      ::entmax::g_trace[(slot)] = clock64();                                                            \
  } while (0)
#define ENTMAX_TRACE_EV(slot) ENTMAX_TRACE_K(0, slot)
// count an event over all CTAs (slots 8100..8191)
#define ENTMAX_TRACE_COUNT(slot) atomicAdd(&::entmax::g_trace[(slot)], 1ull)
#else
#define ENTMAX_TRACE_COUNT(slot) \
  do {                           \
  } while (0)
#define ENTMAX_TRACE_EV(slot) \
  do {                        \
  } while (0)
#define ENTMAX_TRACE_K(kid, slot) \
  do {                            \
  } while (0)
#endif
