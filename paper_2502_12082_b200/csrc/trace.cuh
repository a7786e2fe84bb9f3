// trace.cuh — optional pipeline tracing (diagnostics build only: -DENTMAX_TRACE).  Records
// clock64() timestamps of pipeline events of one CTA (blockIdx == (trace_bx, 0)) into a device
// array that the diagnostics library exports; compiles to nothing in the product build.
#pragma once
#include <cstdint>

#ifdef ENTMAX_TRACE
namespace entmax {
extern __device__ unsigned long long g_trace[8192];
extern __device__ int g_trace_bx;
}
#define ENTMAX_TRACE_EV(slot)                                                                 \
  do {                                                                                        \
    if (blockIdx.x == (unsigned)::entmax::g_trace_bx && blockIdx.y == 0 && (slot) < 8192)       \
      ::entmax::g_trace[(slot)] = clock64();                                                  \
  } while (0)
// count an event over all CTAs (slots 8100..8191)
#define ENTMAX_TRACE_COUNT(slot) atomicAdd(&::entmax::g_trace[(slot)], 1ull)
#else
#define ENTMAX_TRACE_COUNT(slot) \
  do {                           \
  } while (0)
#define ENTMAX_TRACE_EV(slot) \
  do {                        \
  } while (0)
#endif
