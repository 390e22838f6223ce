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

cudaError_t launch_spmv_outer(int s, int rows, int cols, int64_t nnz, const int* row_map,
                              const int* col_entry, const double* values, const double* x,
                              double* z, cudaStream_t st) {
  if (rows <= 0 || s <= 0) return cudaSuccess;
  k_spmv_outer<<<(rows + kOuterRows - 1) / kOuterRows, kOuterRows, 0, st>>>(rows, cols, s, nnz, row_map,
                                                                          col_entry, values, x, z);
  return cudaGetLastError();
}

}  // namespace ep
