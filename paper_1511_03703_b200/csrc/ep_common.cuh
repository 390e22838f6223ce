// Device helpers shared by the enprop_b200 kernels (sm_100a).
//
// Arithmetic rule: every floating-point operation on the hot path goes through
// __dmul_rn / __dadd_rn / __dsub_rn so that no FMA contraction can happen
// (the reference is built with -ffp-contract=off, proj/CMakeLists.txt:14);
// the library is additionally compiled with -fmad=false.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "ep_tilemap.h"

#define EP_DMUL(a, b) __dmul_rn((a), (b))
#define EP_DADD(a, b) __dadd_rn((a), (b))
#define EP_DSUB(a, b) __dsub_rn((a), (b))

// dispatch a runtime ensemble width to a template instantiation
#define EP_DISPATCH_S(s, FN, ...)                 \
  switch (s) {                                    \
    case 1: return FN<1>(__VA_ARGS__);            \
    case 2: return FN<2>(__VA_ARGS__);            \
    case 4: return FN<4>(__VA_ARGS__);            \
    case 8: return FN<8>(__VA_ARGS__);            \
    case 16: return FN<16>(__VA_ARGS__);          \
    case 32: return FN<32>(__VA_ARGS__);          \
    default: return cudaErrorInvalidValue;        \
  }

namespace ep {

// Tuning switches from the environment, read once per process by their call
// sites: an unset OR empty variable means the default (so `VAR=` cannot flip
// a switch silently).
inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

constexpr int kMaxS = 32;
constexpr int kMaxTerms = 64;

template <int V>
struct VecD {
  double v[V];
};

// Streamed once (matrix values, column indices): read-only path, no L1 allocation.
template <int V>
__device__ __forceinline__ VecD<V> ld_stream(const double* p) {
  VecD<V> r;
  if constexpr (V == 1) {
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r.v[0]) : "l"(p));
  } else {
#pragma unroll
    for (int i = 0; i < V; i += 2)
      asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                   : "=d"(r.v[i]), "=d"(r.v[i + 1])
                   : "l"(p + i));
  }
  return r;
}

// Re-used across rows (gathered vectors): default caching.
template <int V>
__device__ __forceinline__ VecD<V> ld_vec(const double* p) {
  VecD<V> r;
  if constexpr (V == 1) {
    r.v[0] = *p;
  } else {
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + i);
      r.v[i] = t.x;
      r.v[i + 1] = t.y;
    }
  }
  return r;
}

template <int V>
__device__ __forceinline__ void st_vec(double* p, const VecD<V>& a) {
  if constexpr (V == 1) {
    *p = a.v[0];
  } else {
#pragma unroll
    for (int i = 0; i < V; i += 2)
      *reinterpret_cast<double2*>(p + i) = make_double2(a.v[i], a.v[i + 1]);
  }
}

__device__ __forceinline__ int ld_stream_i32(const int* p) {
  int r;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// ---- L2 policy for the TMA prefetches (createpolicy) ----------------------
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int V>
__device__ __forceinline__ VecD<V> ld_stream_hint(const double* p, uint64_t pol) {
  VecD<V> r;
  if constexpr (V == 1) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r.v[0]) : "l"(p), "l"(pol));
  } else {
#pragma unroll
    for (int i = 0; i < V; i += 2)
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
          : "=d"(r.v[i]), "=d"(r.v[i + 1])
          : "l"(p + i), "l"(pol));
  }
  return r;
}
__device__ __forceinline__ int ld_stream_i32_hint(const int* p, uint64_t pol) {
  int r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
template <int V>
__device__ __forceinline__ void st_vec_hint(double* p, const VecD<V>& a, uint64_t pol) {
  if constexpr (V == 1) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(a.v[0]), "l"(pol) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < V; i += 2)
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p + i), "d"(a.v[i]),
                   "d"(a.v[i + 1]), "l"(pol)
                   : "memory");
  }
}

// ---- mbarrier + 1D bulk copy (TMA engine, cp.async.bulk) -------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA prefetch of [p, p + bytes) into L2 (bytes a multiple of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- programmatic dependent launch (PDL) -----------------------------------
// Kernels of the CG loop are launched with programmatic stream serialization
// (launch_k): the next kernel's CTAs may be scheduled while this one drains.
// Every such kernel starts with EP_PDL_ENTRY(): allow the dependent grid to be
// scheduled (once all of this grid's CTAs have started, so it never takes SMs
// from them), then wait until the preceding grid has completed and its memory
// is visible -- before any read of its results. Without the launch attribute
// both instructions are no-ops.
#define EP_PDL_ENTRY()                                                  \
  do {                                                                  \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");     \
    asm volatile("griddepcontrol.wait;" ::: "memory");                  \
  } while (0)

// Per-context launch options (ENPROP_OPT_PDL, ENPROP_OPT_SPMV_VARIANT). Every
// C-ABI entry point that launches kernels installs its context's options for
// the duration of the call (ScopedLaunchOpts, ep_internal.h); the launch code
// reads them from this thread-local slot, so concurrent contexts on different
// host threads never see each other's settings.
struct LaunchOpts {
  int pdl = 0;            // PDL default off: -1% on the three-group s = 32 bench, +2-4% single stream
  int spmv_variant = -1;  // warp-SpMV schedule, -1 = auto
};
inline LaunchOpts& launch_opts() {
  thread_local LaunchOpts o;
  return o;
}
inline int pdl_enabled() { return launch_opts().pdl; }

// ENPROP_PDL_MASK (env, tuning): kernel kinds launched with PDL (1 direction,
// 2 SpMV, 4 finalize, 8 update, 16 other); default all
inline int pdl_mask() {
  static int m = env_int("ENPROP_PDL_MASK", 31);
  return m;
}

constexpr int kLaunchCooperative = 64;  // launch_kk kind flag
constexpr int kLaunchUrgent = 128;      // launch_kk kind flag: highest launch priority

// the device's highest (numerically lowest) stream priority, queried once
inline int greatest_priority() {
  static const int v = [] {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) greatest = 0;
    return greatest;
  }();
  return v;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kk(int kind, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  unsigned n = 0;
  if (kind & kLaunchUrgent) {  // pending CTAs of this launch get the next free SM first
    attr[n].id = cudaLaunchAttributePriority;
    attr[n].val.priority = greatest_priority();
    ++n;
  }
  if (pdl_enabled() && (pdl_mask() & kind)) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (kind & kLaunchCooperative) {  // all CTAs co-resident (grid-wide barrier inside)
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace ep
