// trace.cuh -- -DDKV_TRACE builds (`make trace`, tools/trace_bwd.py): clock64 timestamps of
// per-tile events of ONE CTA (chosen at run time), read back through a C-ABI hook.  Each
// translation unit that includes this gets its own buffer.  Compiled out otherwise.
#pragma once

namespace dkv {
enum TraceEv { T_Q_LOAD, T_DO_LOAD, T_ISS_S, T_ISS_DP, T_ISS_DV, T_ISS_DK, T_ISS_DQ, T_C_S, T_C_P, T_C_DP, T_C_DS,
               T_D_DQ, T_D_LD, T_D_END, T_MMA_END, T_EXTRA, T_START, T_KLOAD, T_SISS_END, T_SDONE };
}

#ifdef DKV_TRACE
namespace dkv {
constexpr int kTraceTiles = 256;
constexpr int kTraceEvents = 20;
static __device__ long long g_trace[kTraceEvents * kTraceTiles];
static __device__ int g_trace_cta = -1;
}  // namespace dkv
#define TRACE(ev, i)                                                                                      \
  do {                                                                                                    \
    if (static_cast<int>(blockIdx.x) == ::dkv::g_trace_cta && (i) < ::dkv::kTraceTiles)                   \
      ::dkv::g_trace[(ev) * ::dkv::kTraceTiles + (i)] = clock64();                                        \
  } while (0)
// cta >= 0: arm the trace for that CTA of the next launch (clears); cta < 0: copy it out to dst
#define DKV_TRACE_READ_FN(name)                                                                           \
  extern "C" __attribute__((visibility("default"))) int name(long long* dst, int cta) {                   \
    if (cta >= 0) {                                                                                       \
      static long long zeros[::dkv::kTraceEvents * ::dkv::kTraceTiles] = {};                              \
      cudaMemcpyToSymbol(::dkv::g_trace, zeros, sizeof(zeros));                                           \
      cudaMemcpyToSymbol(::dkv::g_trace_cta, &cta, sizeof(int));                                          \
      return 0;                                                                                           \
    }                                                                                                     \
    return cudaMemcpyFromSymbol(dst, ::dkv::g_trace, sizeof(long long) * ::dkv::kTraceEvents * ::dkv::kTraceTiles) == \
                   cudaSuccess ? 0 : -1;                                                                  \
  }
#else
#define TRACE(ev, i) \
  do {               \
  } while (0)
#define DKV_TRACE_READ_FN(name)
#endif
