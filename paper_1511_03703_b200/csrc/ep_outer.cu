// Sample-major ("outer") ensemble SpMV, spmv_outer (proj/include/enprop/kernels.hpp:38-56)
// on OuterEnsembleMatrix (proj/include/enprop/crs.hpp:138-147): s scalar value
// blocks values[e*nnz + k] over one shared graph, x[e*cols + c], z[e*rows + row].
//
// The reference sweeps the graph once per component. Here a CTA owns a block of
// kOuterRows rows: it stages the block's column indices in shared memory once
// and reuses them for all s components, and for each component streams the
// block's contiguous value range through shared memory with coalesced loads.
// Each thread then forms its row's sum in entry order, ((0 + a_0 x_0) + a_1 x_1)
// + ..., so every component is bitwise the reference's scalar product. Blocks
// whose entries exceed the staging capacity (very long rows of a general CRS)
// read straight from global memory in the same order.
#include "ep_common.cuh"
#include "ep_kernels.h"

namespace ep {

constexpr int kOuterRows = 128;               // rows (= threads) per CTA
constexpr int kOuterCap = kOuterRows * 28;    // staged entries per block

__global__ void __launch_bounds__(kOuterRows) k_spmv_outer(int rows, int cols, int s, int64_t nnz,
                                                           const int* __restrict__ row_map,
                                                           const int* __restrict__ col_entry,
                                                           const double* __restrict__ values,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ z) {
  __shared__ int scol[kOuterCap];
  __shared__ double sval[kOuterCap];
  const int r0 = blockIdx.x * kOuterRows;
  const int r1 = imin(r0 + kOuterRows, rows);
  const int row = r0 + threadIdx.x;
  const int k0 = __ldg(row_map + r0), k1 = __ldg(row_map + r1);
  const int n = k1 - k0;
  const bool staged = n <= kOuterCap;
  int ks = 0, ke = 0;
  if (row < rows) {
    ks = __ldg(row_map + row) - k0;
    ke = __ldg(row_map + row + 1) - k0;
  }
  if (staged)
    for (int i = threadIdx.x; i < n; i += kOuterRows) scol[i] = ld_stream_i32(col_entry + k0 + i);
  for (int e = 0; e < s; ++e) {
    const double* ve = values + (size_t)e * nnz + k0;
    const double* xe = x + (size_t)e * cols;
    if (staged) {
      __syncthreads();  // previous component's values consumed (and scol written)
      for (int i = threadIdx.x; i < n; i += kOuterRows) sval[i] = ld_stream<1>(ve + i).v[0];
      __syncthreads();
    }
    if (row < rows) {
      double sum = 0.0;
      if (staged) {
        for (int k = ks; k < ke; ++k) sum = EP_DADD(sum, EP_DMUL(sval[k], __ldg(xe + scol[k])));
      } else {
        for (int k = ks; k < ke; ++k)
          sum = EP_DADD(sum, EP_DMUL(__ldg(ve + k), __ldg(xe + __ldg(col_entry + k0 + k))));
      }
      z[(size_t)e * rows + row] = sum;
    }
  }
}

// Asynchronous staging (cp.async, LDGSTS): n elements of T from src into shared
// memory at sbase + phase, where phase = src's element offset inside its 16-byte
// granule, so source and destination share the 16-byte phase and every whole
// granule moves with one 16-byte copy; the (at most two) partial granules at the
// ends move element by element. Nothing outside [src, src + n) is read. All of a
// thread's copies are in flight together (no register round trip); the caller
// waits with cp_async_wait_all() + __syncthreads(). Returns the phase.
__device__ __forceinline__ void cp_async16(void* d, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(g) : "memory");
}
template <int B>
__device__ __forceinline__ void cp_async_small(void* d, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(d)), "l"(g), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ int stage_async(T* sbase, const T* src, int n) {
  constexpr int E = 16 / sizeof(T);
  const int ph = (int)((reinterpret_cast<uintptr_t>(src) & 15) / sizeof(T));
  const T* g0 = src - ph;  // 16-byte aligned; only elements >= ph are read
  const int total = ph + n;
  const int ng = (total + E - 1) / E;
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    const int lo = g * E, hi = lo + E;
    if (lo >= ph && hi <= total) {
      cp_async16(sbase + lo, g0 + lo);
    } else {
      for (int i = max(lo, ph); i < min(hi, total); ++i) cp_async_small<sizeof(T)>(sbase + i, g0 + i);
    }
  }
  return ph;
}

// Ensemble-layout SpMV for narrow ensembles (s <= 8): a row's s values are only
// 8s <= 64 bytes, so one thread per (row, sample) walking its row would issue
// strided, uncoalesced loads. Instead a CTA stages its row block's contiguous
// column-index range in shared memory with asynchronous 16-byte copies
// (stage_async), and thread (row, sample e) sums its row in entry order
// (kernels.hpp:15-26, bitwise), reading x through the staged indices and its
// values straight from global memory: a row block's values are one contiguous
// range, so the CTA's value reads touch each 32-byte sector once between them
// and L1 serves the rest; leaving them unstaged cuts the shared memory per CTA
// (s = 1: 22.5 -> 8.2 KB) and raises the resident CTAs (MODE 1, the default;
// A/B in profiles/round1/spmv_small_ab.jsonl). MODE 0 also stages the values,
// MODE 2 only the values. Blocks whose entries exceed the staging capacity read
// everything from global memory in the same order.
template <int S, int NT, int MINB, int MODE>
__global__ void __launch_bounds__(NT, MINB) k_spmv_small(int rows, const int* __restrict__ row_map,
                                                           const int* __restrict__ col_entry,
                                                           const double* __restrict__ values,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ z) {
  // MODE 0: stage indices and values; 1: indices only; 2: values only
  constexpr bool kCols = MODE != 2, kVals = MODE != 1;
  constexpr int RB = NT / S;   // rows per CTA
  constexpr int CAP = RB * 28;  // staged entries
  __shared__ __align__(16) int scol_raw[kCols ? CAP + 4 : 4];
  __shared__ __align__(16) double sval_raw[kVals ? CAP * S + 2 : 2];
  const int r0 = blockIdx.x * RB;
  const int r1 = imin(r0 + RB, rows);
  const int row = r0 + threadIdx.x / S, e = threadIdx.x % S;
  const int k0 = __ldg(row_map + r0), k1 = __ldg(row_map + r1);
  const int n = k1 - k0;
  const bool staged = n <= CAP;
  const int* scol = kCols ? scol_raw : col_entry + k0;
  const double* sval = kVals ? sval_raw : values + (size_t)k0 * S;
  if (staged) {
    if constexpr (kCols) scol += stage_async(scol_raw, col_entry + k0, n);
    if constexpr (kVals) sval += stage_async(sval_raw, values + (size_t)k0 * S, n * S);
  }
  int ks = 0, ke = 0;
  if (row < rows) {
    ks = __ldg(row_map + row) - k0;
    ke = __ldg(row_map + row + 1) - k0;
  }
  if (staged) {
    cp_async_wait_all();
    __syncthreads();
  }
  if (row >= rows) return;
  double sum = 0.0;
  if (staged) {
    for (int k = ks; k < ke; ++k) {
      const int c = kCols ? scol[k] : __ldg(scol + k);
      const double a = kVals ? sval[k * S + e] : __ldg(sval + k * S + e);
      sum = EP_DADD(sum, EP_DMUL(a, __ldg(x + (size_t)c * S + e)));
    }
  } else {
    for (int k = k0 + ks; k < k0 + ke; ++k)
      sum = EP_DADD(sum, EP_DMUL(__ldg(values + (size_t)k * S + e), __ldg(x + (size_t)__ldg(col_entry + k) * S + e)));
  }
  z[(size_t)row * S + e] = sum;
}

// CTA size, register cap and staging mode of the narrow-ensemble SpMV.
// Defaults (A/B at 128^3, tools/small_ab.py, profiles/round1/spmv_small_ab.jsonl):
// 64 threads, indices staged, capped at 64 registers for s = 1 and 48 for s >= 2
// (uncapped, ptxas takes 80-86). A/B switches: ENPROP_SMALL_NT = 64 | 96 | 128,
// ENPROP_SMALL_REGS = 0 (uncapped) | 32 | 48 | 64, every mode at each cap,
// ENPROP_SMALL_STAGE = 0 | 1 | 2.
static int small_nt(int) {
  static const int nt = [] {
    const int v = env_int("ENPROP_SMALL_NT", 0);
    return (v == 96 || v == 128) ? v : 64;
  }();
  return nt;
}
static int small_regs(int s) {
  static const int r = [] {
    const int v = env_int("ENPROP_SMALL_REGS", -1);
    return (v == 0 || v == 32 || v == 48 || v == 64) ? v : -1;
  }();
  // auto: 64 at s = 1 (more resident CTAs shrink L1 below the unstaged value
  // reads' reuse distance: 48 registers cost 30%), 48 at s >= 2 (a row's s
  // values share sectors across threads, so L1 reuse matters less and the
  // extra residency wins: s = 4/8 at 96-98% of HBM vs 80% at 64)
  return r >= 0 ? r : (s == 1 ? 64 : 48);
}

static int small_mode() {
  static const int mode = [] {
    const int v = env_int("ENPROP_SMALL_STAGE", 1);
    return (v == 0 || v == 2) ? v : 1;
  }();
  return mode;
}

template <int S, int NT>
static cudaError_t spmv_small_nt(int rows, const int* row_map, const int* col_entry,
                                 const double* values, const double* x, double* z, cudaStream_t st) {
  constexpr int RB = NT / S;
  if (rows <= 0) return cudaSuccess;
  const int grid = (rows + RB - 1) / RB;
  const int mode = small_mode();
  constexpr int MB = 65536 / (NT * 64);
  switch (small_regs(S) * 4 + mode) {
    case 0: k_spmv_small<S, NT, 1, 0><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 1: k_spmv_small<S, NT, 1, 1><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 2: k_spmv_small<S, NT, 1, 2><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 192: k_spmv_small<S, NT, 65536 / (NT * 48), 0><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 193: k_spmv_small<S, NT, 65536 / (NT * 48), 1><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 194: k_spmv_small<S, NT, 65536 / (NT * 48), 2><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 128: k_spmv_small<S, NT, 65536 / (NT * 32), 0><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 130: k_spmv_small<S, NT, 65536 / (NT * 32), 2><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 129: k_spmv_small<S, NT, 65536 / (NT * 32), 1><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 256: k_spmv_small<S, NT, MB, 0><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    case 258: k_spmv_small<S, NT, MB, 2><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
    default: k_spmv_small<S, NT, MB, 1><<<grid, NT, 0, st>>>(rows, row_map, col_entry, values, x, z); break;
  }
  return cudaGetLastError();
}

template <int S>
static cudaError_t spmv_small_s(int rows, const int* row_map, const int* col_entry,
                                const double* values, const double* x, double* z, cudaStream_t st) {
  switch (small_nt(S)) {
    case 96: return spmv_small_nt<S, 96>(rows, row_map, col_entry, values, x, z, st);
    case 128: return spmv_small_nt<S, 128>(rows, row_map, col_entry, values, x, z, st);
    default: return spmv_small_nt<S, 64>(rows, row_map, col_entry, values, x, z, st);
  }
}

// widest ensemble enprop_spmv sends to k_spmv_small (ENPROP_SMALL_MAX: 8, 16
// or 32; default 16: at 128^3, s = 16 runs at 97% of HBM here vs 90% in the
// warp-per-row k_spmv<16>)
// the configuration launch_spmv_small launches for width s (every (register
// cap, staging mode) pair has its own instantiation: nothing falls back)
void spmv_small_config(int s, int* threads, int* reg_cap, int* stage_mode) {
  if (threads) *threads = small_nt(s);
  if (reg_cap) *reg_cap = small_regs(s);
  if (stage_mode) *stage_mode = small_mode();
}

int spmv_small_max() {
  static const int m = [] {
    const int v = env_int("ENPROP_SMALL_MAX", 16);
    return (v == 8 || v == 32) ? v : 16;
  }();
  return m;
}

cudaError_t launch_spmv_small(int s, int rows, const int* row_map, const int* col_entry,
                              const double* values, const double* x, double* z, cudaStream_t st) {
  switch (s) {
    case 1: return spmv_small_s<1>(rows, row_map, col_entry, values, x, z, st);
    case 2: return spmv_small_s<2>(rows, row_map, col_entry, values, x, z, st);
    case 4: return spmv_small_s<4>(rows, row_map, col_entry, values, x, z, st);
    case 8: return spmv_small_s<8>(rows, row_map, col_entry, values, x, z, st);
    case 16: return spmv_small_s<16>(rows, row_map, col_entry, values, x, z, st);
    case 32: return spmv_small_s<32>(rows, row_map, col_entry, values, x, z, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_spmv_outer(int s, int rows, int cols, int64_t nnz, const int* row_map,
                              const int* col_entry, const double* values, const double* x,
                              double* z, cudaStream_t st) {
  if (rows <= 0 || s <= 0) return cudaSuccess;
  k_spmv_outer<<<(rows + kOuterRows - 1) / kOuterRows, kOuterRows, 0, st>>>(rows, cols, s, nnz, row_map,
                                                                          col_entry, values, x, z);
  return cudaGetLastError();
}

}  // namespace ep
