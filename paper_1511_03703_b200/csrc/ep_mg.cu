// Multigrid preconditioner: the reference's aggregation AMG
// (proj/include/enprop/multigrid.hpp, src/multigrid.cpp) with its V-cycle and
// Chebyshev smoother on the device, bitwise in the reference's operation order.
//
//  * Setup (build_hierarchy, multigrid.hpp:362-396) runs on the host, as in
//    the reference: connection graph (:38-76), greedy root aggregation
//    (multigrid.cpp:5-43), piecewise-constant P and R = P^T (:79-107),
//    Galerkin coarse operator in the reference's accumulation order
//    (:114-160), diagonal. This file is compiled with -ffp-contract=off on
//    the host. The power-iteration lambda_max per component (:170-206) runs
//    on the device from the uploaded level (device_power_lambda_max: the
//    same operations, 1.8 s -> milliseconds at 32^3, s = 32).
//  * The coarsest operator is factored by dense LU with partial pivoting per
//    component ON THE DEVICE (DenseLuSolver::factor, :297-317): blocked in
//    32-column panels (a 4-CTA cluster per component factors a panel) with
//    the unblocked right-looking algorithm's per-element operation order (pivot = first maximum,
//    full-row swaps, multiplier then trailing update), so the factors are the
//    reference's bits. The reference's own host LU makes >= 64^3 infeasible
//    (the Dirichlet rows stay singleton aggregates: >= 2(n+1)^2 coarse rows).
//  * V-cycle (:402-425) on the device: Chebyshev (:232-260) with per-lane
//    recurrence coefficients precomputed on the host in the reference's order,
//    residual, restriction as an SpMV with R (bitwise launch_spmv), zero coarse
//    guess, recursion, prolongation x += 1.0 * z[aggregate], post-smoothing.
//    Coarse solve (:269-290): pivot swaps, forward substitution as a column
//    sweep (each row still subtracts its terms in increasing column order),
//    back substitution as one chain per component (its row order leaves no
//    parallelism: row r's first term needs y[r+1]).
//  * pcg_solve with MgPreconditioner (pcg.hpp:52-103): host-driven loop, the
//    reference's serial dot order through the chain kernel (ep_chain.cu);
//    coupled (one decision) or uncoupled (per-lane scalars, converged lanes
//    frozen), matching s x pcg_solve<double> on extracted components.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "enprop_b200.h"
#include "ep_common.cuh"
#include "ep_internal.h"
#include "ep_kernels.h"

using namespace ep;
using namespace ep_internal;

namespace {

// ============================================================== device kernels
// Chebyshev first step (multigrid.hpp:244-246): r = b - tmp; p = (r / diag) / theta; x += p
template <int S>
__global__ void k_cheb_first(int64_t n, const double* __restrict__ b, const double* __restrict__ tmp,
                             const double* __restrict__ diag, const double* __restrict__ theta,
                             double* __restrict__ r, double* __restrict__ p, double* __restrict__ x) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int e = (int)(g % S);
  const double rv = EP_DSUB(b[g], tmp[g]);
  const double pv = __ddiv_rn(__ddiv_rn(rv, diag[g]), theta[e]);
  r[g] = rv;
  p[g] = pv;
  x[g] = EP_DADD(x[g], pv);
}

// Chebyshev step k (:248-257): r -= tmp; p = pc*p + zc*(r / diag); x += p
template <int S>
__global__ void k_cheb_next(int64_t n, const double* __restrict__ tmp, const double* __restrict__ diag,
                            const double* __restrict__ pc, const double* __restrict__ zc,
                            double* __restrict__ r, double* __restrict__ p, double* __restrict__ x) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int e = (int)(g % S);
  const double rv = EP_DSUB(r[g], tmp[g]);
  const double pv = EP_DADD(EP_DMUL(pc[e], p[g]), EP_DMUL(zc[e], __ddiv_rn(rv, diag[g])));
  r[g] = rv;
  p[g] = pv;
  x[g] = EP_DADD(x[g], pv);
}

// V-cycle residual (:411-412): tmp = b - tmp
template <int S>
__global__ void k_sub_from(int64_t n, const double* __restrict__ b, double* __restrict__ tmp) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n * S) tmp[g] = EP_DSUB(b[g], tmp[g]);
}

// prolongation (:418-420): x[row] += P.values[k] * z[P.col[k]] with one entry 1.0 per row
template <int S>
__global__ void k_prolong(int64_t n, const int* __restrict__ agg, const double* __restrict__ z,
                          double* __restrict__ x) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int64_t row = g / S;
  const int e = (int)(g - row * S);
  x[g] = EP_DADD(x[g], EP_DMUL(1.0, z[(int64_t)agg[row] * S + e]));
}

// masked axpby for the MG-PCG loop: y = a*x + 1.0*y on active lanes (pcg.hpp:94-95)
template <int S>
__global__ void k_axpy_masked(int64_t n, const double* __restrict__ a, const int* __restrict__ act,
                              const double* __restrict__ x, double* __restrict__ y) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int e = (int)(g % S);
  if (act[e]) y[g] = EP_DADD(EP_DMUL(a[e], x[g]), EP_DMUL(1.0, y[g]));
}

// p = 1.0*z + beta*p on active lanes (pcg.hpp:101)
template <int S>
__global__ void k_direction_masked(int64_t n, const double* __restrict__ beta, const int* __restrict__ act,
                                   const double* __restrict__ z, double* __restrict__ p) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int e = (int)(g % S);
  if (act[e]) p[g] = EP_DADD(EP_DMUL(1.0, z[g]), EP_DMUL(beta[e], p[g]));
}

// Dense LU with partial pivoting per component (DenseLuSolver::factor,
// multigrid.hpp:297-317): lu is [s][n][n] row-major, piv [s][n]. Pivot row = the
// first row with the largest |lu[row][k]| (strict '>' in row order).
constexpr int kLuThreads = 1024;

// A cluster of kLuCluster CTAs factors one component, so each step's pivot
// search, row swap and trailing update are spread over kLuCluster SMs (a
// single CTA per component was bound by one SM's memory pipe: 2.2 s for
// 32 x 2179^2). The cluster combines the CTAs' pivot candidates through
// distributed shared memory; barriers separate the phases of a step, and
// every element sees the reference's operations in the reference's order.
constexpr int kLuCluster = 4;

__global__ void __cluster_dims__(kLuCluster, 1, 1) __launch_bounds__(kLuThreads)
    k_lu_factor(int n, int k0, int k1, double* __restrict__ lu_all, int* __restrict__ piv_all,
                int* __restrict__ singular) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const int comp = blockIdx.x / kLuCluster;
  double* lu = lu_all + (size_t)comp * n * n;
  int* piv = piv_all + (size_t)comp * n;
  __shared__ double s_best[kLuThreads / 32];
  __shared__ int s_row[kLuThreads / 32];
  __shared__ double c_best;  // this CTA's pivot candidate, read by the whole cluster
  __shared__ int c_row;
  __shared__ int s_pivot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int T = kLuCluster * kLuThreads;          // threads of the cluster
  constexpr int W = kLuCluster * (kLuThreads / 32);   // warps of the cluster
  const int gt = q * kLuThreads + tid, gw = q * (kLuThreads / 32) + warp;
  for (int k = k0; k < k1; ++k) {  // the panel's columns [k0, k1)
    // pivot: the first row with the largest |lu[row][k]|, row >= k (each
    // thread scans its rows in order with '>', combines keep the smaller row)
    double best = -1.0;
    int brow = n;
    for (int row = k + gt; row < n; row += T) {
      const double c = fabs(lu[(size_t)row * n + k]);
      if (c > best) {
        best = c;
        brow = row;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const int orow = __shfl_down_sync(0xffffffffu, brow, o);
      if (ob > best || (ob == best && orow < brow)) {
        best = ob;
        brow = orow;
      }
    }
    if (lane == 0) {
      s_best[warp] = best;
      s_row[warp] = brow;
    }
    __syncthreads();
    if (tid == 0) {
      double bb = s_best[0];
      int r = s_row[0];
      for (int w = 1; w < kLuThreads / 32; ++w)
        if (s_best[w] > bb || (s_best[w] == bb && s_row[w] < r)) {
          bb = s_best[w];
          r = s_row[w];
        }
      c_best = bb;
      c_row = r;
    }
    cluster.sync();  // candidates visible to the cluster
    if (tid == 0) {
      double bb = -1.0;
      int r = n;
      for (int j = 0; j < kLuCluster; ++j) {
        const double bj = *cluster.map_shared_rank(&c_best, j);
        const int rj = *cluster.map_shared_rank(&c_row, j);
        if (bj > bb || (bj == bb && rj < r)) {
          bb = bj;
          r = rj;
        }
      }
      if (q == 0) {
        if (bb == 0.0) atomicExch(singular, 1);
        piv[k] = r < n ? r : k;
      }
      s_pivot = r < n ? r : k;
    }
    __syncthreads();
    const int pr = s_pivot;
    if (pr != k)  // the swap within the panel's columns (k_lu_swaps does the rest)
      for (int col = k0 + gt; col < k1; col += T) {
        const double t = lu[(size_t)k * n + col];
        lu[(size_t)k * n + col] = lu[(size_t)pr * n + col];
        lu[(size_t)pr * n + col] = t;
      }
    cluster.sync();  // row k final for this step; the candidates were read
    // multipliers, then each row's trailing update (a warp per row):
    // mult = lu[row][k] * inv_pivot; lu[row][col] -= mult * lu[k][col]
    const double inv = __ddiv_rn(1.0, lu[(size_t)k * n + k]);
    for (int row = k + 1 + gw; row < n; row += W) {
      double mult = 0.0;
      if (lane == 0) {
        mult = EP_DMUL(lu[(size_t)row * n + k], inv);
        lu[(size_t)row * n + k] = mult;
      }
      mult = __shfl_sync(0xffffffffu, mult, 0);
      double* lrow = lu + (size_t)row * n;
      const double* krow = lu + (size_t)k * n;
      for (int col = k + 1 + lane; col < k1; col += 32) lrow[col] = EP_DSUB(lrow[col], EP_DMUL(mult, krow[col]));
    }
    cluster.sync();  // step complete: the next pivot search reads column k + 1
  }
}

// Blocked LU with the unblocked algorithm's bits. After the panel [k0, k1) is
// factored (k_lu_factor on its columns), the other columns receive the
// panel's row swaps in order (k_lu_swaps), the panel rows of the trailing
// columns their updates from the panel steps (k_lu_u12), and the trailing
// rows theirs (k_lu_trailing). Every element still sees each step's update
// lu[i][j] -= lu[i][t] * lu[t][j] one at a time in increasing t, with the
// multiplier and pivot row the unblocked algorithm uses (swaps move whole
// rows, multipliers included), so the factors are the reference's.
constexpr int kLuPanel = 32;

__global__ void k_lu_swaps(int n, int k0, int k1, double* __restrict__ lu_all, const int* __restrict__ piv_all) {
  const int comp = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (j >= k0 && j < k1)) return;
  double* lu = lu_all + (size_t)comp * n * n;
  const int* piv = piv_all + (size_t)comp * n;
  for (int k = k0; k < k1; ++k) {
    const int p = piv[k];
    if (p != k) {
      const double t = lu[(size_t)k * n + j];
      lu[(size_t)k * n + j] = lu[(size_t)p * n + j];
      lu[(size_t)p * n + j] = t;
    }
  }
}

// rows k0..k1-1 of column j >= k1: u[r] -= lu[r][t] * u[t] for t = k0..r-1
__global__ void __launch_bounds__(128) k_lu_u12(int n, int k0, int k1, double* __restrict__ lu_all) {
  __shared__ double L[kLuPanel][kLuPanel];
  const int comp = blockIdx.y;
  double* lu = lu_all + (size_t)comp * n * n;
  const int bw = k1 - k0;
  for (int i = threadIdx.x; i < bw * bw; i += blockDim.x) L[i / bw][i % bw] = lu[(size_t)(k0 + i / bw) * n + k0 + i % bw];
  __syncthreads();
  const int j = k1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double u[kLuPanel];
#pragma unroll
  for (int r = 0; r < kLuPanel; ++r) u[r] = r < bw ? lu[(size_t)(k0 + r) * n + j] : 0.0;
#pragma unroll
  for (int r = 1; r < kLuPanel; ++r) {
    if (r < bw) {
      double acc = u[r];
#pragma unroll
      for (int t = 0; t < r; ++t) acc = EP_DSUB(acc, EP_DMUL(L[r][t], u[t]));
      u[r] = acc;
    }
  }
#pragma unroll
  for (int r = 1; r < kLuPanel; ++r)
    if (r < bw) lu[(size_t)(k0 + r) * n + j] = u[r];
}

// trailing rows and columns >= k1: lu[i][j] -= lu[i][t] * lu[t][j], t = k0..k1-1
// in order; 64 x 64 output tiles, 256 threads, 4 x 4 outputs each
constexpr int kLuTile = 64;
__global__ void __launch_bounds__(256) k_lu_trailing(int n, int k0, int k1, double* __restrict__ lu_all) {
  __shared__ double Ls[kLuTile][kLuPanel + 1];
  __shared__ double Us[kLuPanel][kLuTile];
  const int comp = blockIdx.z;
  double* lu = lu_all + (size_t)comp * n * n;
  const int bw = k1 - k0;
  const int i0 = k1 + blockIdx.y * kLuTile, j0 = k1 + blockIdx.x * kLuTile;
  for (int idx = threadIdx.x; idx < kLuTile * kLuPanel; idx += blockDim.x) {
    const int r = idx / kLuPanel, t = idx % kLuPanel;
    Ls[r][t] = (i0 + r < n && t < bw) ? lu[(size_t)(i0 + r) * n + k0 + t] : 0.0;
    const int tt = idx / kLuTile, c = idx % kLuTile;
    Us[tt][c] = (j0 + c < n && tt < bw) ? lu[(size_t)(k0 + tt) * n + j0 + c] : 0.0;
  }
  __syncthreads();
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      acc[a][b] = (i < n && j < n) ? lu[(size_t)i * n + j] : 0.0;
    }
  for (int t = 0; t < bw; ++t)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double l = Ls[ty + 16 * a][t];
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = EP_DSUB(acc[a][b], EP_DMUL(l, Us[t][tx + 16 * b]));
    }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty + 16 * a, j = j0 + tx + 16 * b;
      if (i < n && j < n) lu[(size_t)i * n + j] = acc[a][b];
    }
}

// DenseLuSolver::solve (multigrid.hpp:269-290) of one component per CTA:
// x[row][e] from b[row][e] (ensemble layout), lu [s][n][n], luT [s][n][n]
// (column-major copy for the forward sweep), piv [s][n]; y in shared memory.
template <int S>
__global__ void __launch_bounds__(kLuThreads) k_lu_solve(int n, const double* __restrict__ lu_all,
                                                         const double* __restrict__ luT_all,
                                                         const int* __restrict__ piv_all,
                                                         const double* __restrict__ b, double* __restrict__ x) {
  extern __shared__ double y[];
  const int e = blockIdx.x;
  const double* lu = lu_all + (size_t)e * n * n;
  const double* luT = luT_all + (size_t)e * n * n;
  const int* piv = piv_all + (size_t)e * n;
  const int tid = threadIdx.x;
  for (int row = tid; row < n; row += kLuThreads) y[row] = b[(size_t)row * S + e];
  __syncthreads();
  if (tid == 0)  // row swaps in order k = 0..n-1 (:276-277)
    for (int k = 0; k < n; ++k)
      if (piv[k] != k) {
        const double t = y[k];
        y[k] = y[piv[k]];
        y[piv[k]] = t;
      }
  __syncthreads();
  // forward (:278-282): acc = y[row]; acc -= lu[row][col]*y[col], col ascending;
  // as a column sweep every row still applies its columns in ascending order
  for (int col = 0; col + 1 < n; ++col) {
    const double yc = y[col];
    for (int row = col + 1 + tid; row < n; row += kLuThreads)
      y[row] = EP_DSUB(y[row], EP_DMUL(luT[(size_t)col * n + row], yc));
    __syncthreads();
  }
  // backward (:283-287): acc = y[row]; acc -= lu[row][col]*y[col] for col =
  // row+1..n-1; y[row] = acc / lu[row][row]. Row r's first term needs y[r+1],
  // so the rows run one after another on thread 0, whose chain reads its
  // products from shared memory: the other threads form row r-1's products
  // lu[r-1][c]*y[c] for c >= r+1 (all final) while row r's chain runs, and
  // thread 0 forms each row's first, dependent product itself. Products,
  // subtractions and their column order are the reference's.
  double* pb[2] = {y + n, y + 2 * n};  // products of rows of even / odd index
  for (int r = n - 1; r >= 0; --r) {
    if (tid == 0) {
      const double* lr = lu + (size_t)r * n;
      const double* cur = pb[r & 1];  // lu[r][c]*y[c] for c >= r+2
      double acc = y[r];
      if (r + 1 < n) acc = EP_DSUB(acc, EP_DMUL(lr[r + 1], y[r + 1]));
      for (int c = r + 2; c < n; ++c) acc = EP_DSUB(acc, cur[c]);
      y[r] = __ddiv_rn(acc, lr[r]);
    } else if (r >= 1) {
      const double* lq = lu + (size_t)(r - 1) * n;
      double* nxt = pb[(r - 1) & 1];
      for (int c = r + 1 + (tid - 1); c < n; c += kLuThreads - 1) nxt[c] = EP_DMUL(lq[c], y[c]);
    }
    __syncthreads();
  }
  __syncthreads();
  for (int row = tid; row < n; row += kLuThreads) x[(size_t)row * S + e] = y[row];
}

// dense[e][row][col] = values[k][e] for the entries k of row (thread = (row, e))
__global__ void k_dense_scatter(int n, int s, const int* __restrict__ rm, const int* __restrict__ ce,
                                const double* __restrict__ vals, double* __restrict__ dense) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)n * s) return;
  const int row = (int)(g / s), e = (int)(g % s);
  double* d = dense + (size_t)e * n * n + (size_t)row * n;
  for (int k = rm[row]; k < rm[row + 1]; ++k) d[ce[k]] = vals[(size_t)k * s + e];
}

__global__ void k_transpose_sq(int n, const double* __restrict__ a, double* __restrict__ t) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nn = (int64_t)n * n;
  if (g >= nn * gridDim.y) return;
  const int64_t c = blockIdx.y;
  const int64_t i = g / n, j = g % n;
  if (g < nn) t[c * nn + j * n + i] = a[c * nn + i * n + j];
}

inline int blocks_for(int64_t work) { return (int)((work + 255) / 256); }

// k_lu_solve's shared memory: y and the two product buffers of the back substitution
inline size_t lu_solve_smem(int n) { return (size_t)3 * n * sizeof(double); }

cudaError_t lu_solve_smem_optin(int s, size_t bytes) {
  switch (s) {
    case 1: return cudaFuncSetAttribute(k_lu_solve<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    case 2: return cudaFuncSetAttribute(k_lu_solve<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    case 4: return cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    case 8: return cudaFuncSetAttribute(k_lu_solve<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    case 16: return cudaFuncSetAttribute(k_lu_solve<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    case 32: return cudaFuncSetAttribute(k_lu_solve<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    default: return cudaErrorInvalidValue;
  }
}

#define EP_MG_DISPATCH(s, KER, grid, block, smem, st, ...) \
  switch (s) {                                               \
    case 1: KER<1><<<grid, block, smem, st>>>(__VA_ARGS__); break;   \
    case 2: KER<2><<<grid, block, smem, st>>>(__VA_ARGS__); break;   \
    case 4: KER<4><<<grid, block, smem, st>>>(__VA_ARGS__); break;   \
    case 8: KER<8><<<grid, block, smem, st>>>(__VA_ARGS__); break;   \
    case 16: KER<16><<<grid, block, smem, st>>>(__VA_ARGS__); break; \
    case 32: KER<32><<<grid, block, smem, st>>>(__VA_ARGS__); break; \
    default: break;                                          \
  }

// Power iteration on the device (power_lambda_max, multigrid.hpp:170-206):
// w /= diag elementwise, and per lane the max |w| (exact and order-free, so a
// block-level shared-memory max then one global atomic per lane; the bits of a
// non-negative double order like its value)
template <int S>
__global__ void __launch_bounds__(256) k_pow_div_absmax(int64_t n, double* __restrict__ w,
                                                        const double* __restrict__ diag,
                                                        unsigned long long* __restrict__ maxbits) {
  __shared__ unsigned long long smax[S];
  if (threadIdx.x < S) smax[threadIdx.x] = 0ull;
  __syncthreads();
  const int e = threadIdx.x % S;  // blockDim and the stride are multiples of S
  unsigned long long m = 0ull;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n * S; g += (int64_t)gridDim.x * blockDim.x) {
    const double q = __ddiv_rn(w[g], diag[g]);
    w[g] = q;
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(q));
    m = b > m ? b : m;
  }
  atomicMax(&smax[e], m);
  __syncthreads();
  if (threadIdx.x < S) atomicMax(&maxbits[threadIdx.x], smax[threadIdx.x]);
}

// v = w / scale per lane; a lane whose scale is zero sets *collapsed
template <int S>
__global__ void __launch_bounds__(256) k_pow_scale(int64_t n, const double* __restrict__ w,
                                                   const unsigned long long* __restrict__ maxbits,
                                                   double* __restrict__ v, int* __restrict__ collapsed) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < S && maxbits[g] == 0ull) *collapsed = 1;
  if (g >= n * S) return;
  v[g] = __ddiv_rn(w[g], __longlong_as_double((long long)maxbits[g % S]));
}

template <int S>
__global__ void k_fill_one(int64_t n, double* __restrict__ v) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n) v[g] = 1.0;
}

// ================================================================= host setup
struct HostCrs {
  int rows = 0, cols = 0;
  std::vector<int> rm, ce;
  std::vector<double> v;  // [nnz][s]
};

int find_entry(const HostCrs& a, int row, int col) {
  const auto b = a.ce.begin() + a.rm[row], e = a.ce.begin() + a.rm[row + 1];
  const auto it = std::lower_bound(b, e, col);
  return (it == e || *it != col) ? -1 : (int)(it - a.ce.begin());
}

// connection_graph (multigrid.hpp:38-76)
void connection_graph(const HostCrs& a, int s, std::vector<int>& grm, std::vector<int>& gce) {
  std::vector<char> keep(a.ce.size(), 0);
  for (int row = 0; row < a.rows; ++row)
    for (int k = a.rm[row]; k < a.rm[row + 1]; ++k) {
      if (keep[k]) continue;
      bool nonzero = false;
      for (int e = 0; e < s && !nonzero; ++e) nonzero = a.v[(size_t)k * s + e] != 0.0;
      if (!nonzero) continue;
      keep[k] = 1;
      const int col = a.ce[k];
      if (col == row || col >= a.rows) continue;
      const int t = find_entry(a, col, row);
      if (t >= 0) keep[t] = 1;
    }
  grm.assign(a.rows + 1, 0);
  for (int row = 0; row < a.rows; ++row) {
    int c = 0;
    for (int k = a.rm[row]; k < a.rm[row + 1]; ++k) c += keep[k];
    grm[row + 1] = grm[row] + c;
  }
  gce.clear();
  gce.reserve(grm.back());
  for (int row = 0; row < a.rows; ++row)
    for (int k = a.rm[row]; k < a.rm[row + 1]; ++k)
      if (keep[k]) gce.push_back(a.ce[k]);
}

// aggregate_graph (src/multigrid.cpp:5-43)
int aggregate_graph(int rows, const std::vector<int>& grm, const std::vector<int>& gce, std::vector<int>& agg) {
  agg.assign(rows, -1);
  int next_id = 0;
  for (int row = 0; row < rows; ++row) {
    if (agg[row] != -1) continue;
    bool absorbed_any = false;
    int smallest = -1;
    for (int k = grm[row]; k < grm[row + 1]; ++k) {
      const int col = gce[k];
      if (col == row) continue;
      if (agg[col] == -1) {
        if (!absorbed_any) {
          absorbed_any = true;
          agg[row] = next_id;
        }
        agg[col] = next_id;
      } else if (smallest == -1 || agg[col] < smallest) {
        smallest = agg[col];
      }
    }
    if (absorbed_any) ++next_id;
    else if (smallest != -1) agg[row] = smallest;
    else agg[row] = next_id++;
  }
  return next_id;
}

// galerkin_coarse (multigrid.hpp:114-160), per component in the reference's order
HostCrs galerkin_coarse(const HostCrs& a, int s, const std::vector<int>& agg, int nc) {
  std::vector<int> gmap(nc + 1, 0), grows(a.rows);
  for (int i = 0; i < a.rows; ++i) ++gmap[agg[i] + 1];
  for (int g = 0; g < nc; ++g) gmap[g + 1] += gmap[g];
  {
    std::vector<int> at(gmap.begin(), gmap.end() - 1);
    for (int i = 0; i < a.rows; ++i) grows[at[agg[i]]++] = i;
  }
  HostCrs c;
  c.rows = c.cols = nc;
  c.rm.assign(nc + 1, 0);
  std::vector<double> accum((size_t)nc * s, 0.0);
  std::vector<int> touched;
  std::vector<char> seen(nc, 0);
  for (int big = 0; big < nc; ++big) {
    touched.clear();
    for (int idx = gmap[big]; idx < gmap[big + 1]; ++idx) {
      const int i = grows[idx];
      for (int k = a.rm[i]; k < a.rm[i + 1]; ++k) {
        const int cj = agg[a.ce[k]];
        double* acc = &accum[(size_t)cj * s];
        const double* v = &a.v[(size_t)k * s];
        if (!seen[cj]) {
          seen[cj] = 1;
          touched.push_back(cj);
          for (int e = 0; e < s; ++e) acc[e] = v[e];
        } else {
          for (int e = 0; e < s; ++e) acc[e] += v[e];
        }
      }
    }
    std::sort(touched.begin(), touched.end());
    for (int cj : touched) {
      c.ce.push_back(cj);
      for (int e = 0; e < s; ++e) c.v.push_back(accum[(size_t)cj * s + e]);
      seen[cj] = 0;
    }
    c.rm[big + 1] = (int)c.ce.size();
  }
  return c;
}

// diagonal_of (crs.hpp:124-132)
std::vector<double> diagonal_of(const HostCrs& a, int s) {
  std::vector<double> d((size_t)a.rows * s, 0.0);
  for (int row = 0; row < a.rows; ++row) {
    const int k = find_entry(a, row, row);
    if (k >= 0)
      for (int e = 0; e < s; ++e) d[(size_t)row * s + e] = a.v[(size_t)k * s + e];
  }
  return d;
}

struct LevelDev {
  int rows = 0, coarse_rows = 0;
  int64_t nnz = 0, rnnz = 0;
  int *rm = nullptr, *ce = nullptr, *rrm = nullptr, *rce = nullptr, *agg = nullptr;
  double *vals = nullptr, *rvals = nullptr, *diag = nullptr;
  double* cheb = nullptr;  // [theta | pc_2 | zc_2 | pc_3 | zc_3 ...] x s
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *tmp = nullptr;
  std::vector<double> lmax;
};

}  // namespace

struct enprop_mg {
  enprop_ctx* ctx = nullptr;
  int s = 0;
  enprop_mg_options opt{};
  std::vector<LevelDev> lv;  // lv.back() is the coarsest (dense LU)
  int coarse_n = 0;
  double *lu = nullptr, *luT = nullptr;
  int* piv = nullptr;
  // PCG workspace (level-0 sized)
  double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr, *coef = nullptr, *lanes = nullptr;
  int* act = nullptr;
  CgState* fin_state = nullptr;
};

namespace {

void free_level(LevelDev& l) {
  for (void* q : {(void*)l.rm, (void*)l.ce, (void*)l.rrm, (void*)l.rce, (void*)l.agg, (void*)l.vals,
                  (void*)l.rvals, (void*)l.diag, (void*)l.cheb, (void*)l.b, (void*)l.x, (void*)l.r,
                  (void*)l.p, (void*)l.tmp})
    if (q) cudaFree(q);
  l = LevelDev{};
}

template <class T>
int upload(T** dst, const std::vector<T>& src) {
  EP_CUDA(cudaMalloc(dst, std::max<size_t>(src.size(), 1) * sizeof(T)));
  if (!src.empty()) EP_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return ENPROP_OK;
}

// Chebyshev recurrence scalars per lane (multigrid.hpp:236-256), in the
// reference's Ensemble operation order
std::vector<double> cheb_coeffs(const std::vector<double>& lmax, int s, const enprop_mg_options& o) {
  const int deg = o.chebyshev_degree;
  std::vector<double> out((size_t)(1 + 2 * std::max(deg - 1, 0)) * s);
  for (int e = 0; e < s; ++e) {
    const double top = lmax[e] * o.eigenvalue_boost;
    const double bottom = lmax[e] / o.eigenvalue_ratio;
    const double theta = (top + bottom) * 0.5;
    const double delta = (top - bottom) * 0.5;
    const double sigma = theta / delta;
    double rho = 1.0 / sigma;
    out[e] = theta;
    for (int k = 2; k <= deg; ++k) {
      const double rho_next = 1.0 / (2.0 * sigma - rho);
      out[(size_t)(1 + 2 * (k - 2)) * s + e] = rho_next * rho;
      out[(size_t)(2 + 2 * (k - 2)) * s + e] = 2.0 * rho_next / delta;
      rho = rho_next;
    }
  }
  return out;
}

cudaError_t spmv_level(enprop_mg* h, int s, int rows, int cols, const int* rm, const int* ce,
                       const double* v, const double* x, double* z) {
  h->ctx->launches += 1;
  if (s <= spmv_small_max()) return launch_spmv_small(s, rows, rm, ce, v, x, z, h->ctx->stream);
  return launch_spmv(s, rows, rm, ce, v, x, z, false, h->ctx->stream);
}

// power_lambda_max (multigrid.hpp:170-206) on the device, per component:
// every step is the reference's operation (the level SpMV is the bitwise
// kernel, w / diag and w / scale are IEEE divisions, the final Rayleigh
// quotient's dots are reference-order chains), so lmax is the reference's.
// Status 2: an iteration collapsed to zero (the reference's domain_error).
// Uses the level's r (v) and tmp (w) vectors.
int device_power_lambda_max(enprop_mg* h, LevelDev& l, int iterations, std::vector<double>& lmax, int& status) {
  const int s = h->s;
  const int64_t n = l.rows;
  cudaStream_t st = h->ctx->stream;
  status = 0;
  lmax.assign(s, 1.0);
  if (iterations <= 0) return ENPROP_OK;
  double* v = l.r;
  double* w = l.tmp;
  // scratch: per-lane max bits [s], two lane outputs [2][s + 1], the collapse flag
  double* scratch = nullptr;
  EP_CUDA(cudaMalloc(&scratch, (kMaxS + 2 * (kMaxS + 1) + 1) * sizeof(double)));
  struct FreeOnExit {
    double* q;
    ~FreeOnExit() { cudaFree(q); }
  } free_scratch{scratch};
  unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(scratch);
  double* lanes = scratch + kMaxS;
  int* collapsed = reinterpret_cast<int*>(scratch + kMaxS + 2 * (kMaxS + 1));
  EP_MG_DISPATCH(s, k_fill_one, blocks_for(n * s), 256, 0, st, n * s, v);
  EP_CUDA(cudaMemsetAsync(collapsed, 0, sizeof(int), st));
  const int grid = std::max(1, std::min(4 * 148, (int)((n * s + 255) / 256)));
  for (int it = 0; it < iterations; ++it) {
    EP_CUDA(spmv_level(h, s, l.rows, l.rows, l.rm, l.ce, l.vals, v, w));
    EP_CUDA(cudaMemsetAsync(maxbits, 0, s * sizeof(unsigned long long), st));
    EP_MG_DISPATCH(s, k_pow_div_absmax, grid, 256, 0, st, n, w, l.diag, maxbits);
    h->ctx->launches += 1;
    if (it + 1 == iterations) break;
    EP_MG_DISPATCH(s, k_pow_scale, blocks_for(n * s), 256, 0, st, n, w, maxbits, v, collapsed);
    h->ctx->launches += 1;
  }
  FinArgs f{};
  f.phase = kPhaseNone;
  f.lanes_out = lanes;
  EP_CUDA(launch_chain(s, l.rows, v, w, kChainProduct, f, st));  // num = v . w
  f.lanes_out = lanes + (s + 1);
  EP_CUDA(launch_chain(s, l.rows, v, nullptr, kChainSquare, f, st));  // den = v . v
  h->ctx->launches += 2;
  std::vector<double> hb(2 * (s + 1));
  int hc = 0;
  EP_CUDA(cudaMemcpyAsync(hb.data(), lanes, hb.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  EP_CUDA(cudaMemcpyAsync(&hc, collapsed, sizeof(int), cudaMemcpyDeviceToHost, st));
  EP_CUDA(cudaStreamSynchronize(st));
  if (hc) {
    status = 2;
    return ENPROP_OK;
  }
  for (int e = 0; e < s; ++e) lmax[e] = hb[e] / hb[(s + 1) + e];
  return ENPROP_OK;
}

int chebyshev(enprop_mg* h, LevelDev& l, const double* b, double* x) {
  const int s = h->s;
  cudaStream_t st = h->ctx->stream;
  const int64_t n = l.rows;
  EP_CUDA(spmv_level(h, s, l.rows, l.rows, l.rm, l.ce, l.vals, x, l.tmp));
  EP_MG_DISPATCH(s, k_cheb_first, blocks_for(n * s), 256, 0, st, n, b, l.tmp, l.diag, l.cheb, l.r, l.p, x);
  h->ctx->launches += 1;
  for (int k = 2; k <= h->opt.chebyshev_degree; ++k) {
    EP_CUDA(spmv_level(h, s, l.rows, l.rows, l.rm, l.ce, l.vals, l.p, l.tmp));
    const double* pc = l.cheb + (size_t)(1 + 2 * (k - 2)) * s;
    const double* zc = l.cheb + (size_t)(2 + 2 * (k - 2)) * s;
    EP_MG_DISPATCH(s, k_cheb_next, blocks_for(n * s), 256, 0, st, n, l.tmp, l.diag, pc, zc, l.r, l.p, x);
    h->ctx->launches += 1;
  }
  return cudaGetLastError() == cudaSuccess ? ENPROP_OK : cuda_fail(cudaGetLastError(), "chebyshev");
}

int coarse_solve(enprop_mg* h, const double* b, double* x) {
  const int n = h->coarse_n, s = h->s;
  const size_t smem = lu_solve_smem(n);
  EP_MG_DISPATCH(s, k_lu_solve, s, kLuThreads, smem, h->ctx->stream, n, h->lu, h->luT, h->piv, b, x);
  h->ctx->launches += 1;
  EP_CUDA(cudaGetLastError());
  return ENPROP_OK;
}

// vcycle (multigrid.hpp:402-425) on level k: b, x device vectors of that level
int vcycle(enprop_mg* h, int k, const double* b, double* x) {
  if (k + 1 == (int)h->lv.size()) return coarse_solve(h, b, x);
  LevelDev& l = h->lv[k];
  LevelDev& c = h->lv[k + 1];
  const int s = h->s;
  cudaStream_t st = h->ctx->stream;
  int rc = chebyshev(h, l, b, x);
  if (rc) return rc;
  EP_CUDA(spmv_level(h, s, l.rows, l.rows, l.rm, l.ce, l.vals, x, l.tmp));
  EP_MG_DISPATCH(s, k_sub_from, blocks_for((int64_t)l.rows * s), 256, 0, st, (int64_t)l.rows, b, l.tmp);
  EP_CUDA(spmv_level(h, s, l.coarse_rows, l.rows, l.rrm, l.rce, l.rvals, l.tmp, c.b));  // rc = R tmp
  EP_CUDA(cudaMemsetAsync(c.x, 0, (size_t)c.rows * s * sizeof(double), st));        // z = 0
  h->ctx->launches += 1;
  if ((rc = vcycle(h, k + 1, c.b, c.x))) return rc;
  EP_MG_DISPATCH(s, k_prolong, blocks_for((int64_t)l.rows * s), 256, 0, st, (int64_t)l.rows, l.agg, c.x, x);
  h->ctx->launches += 1;
  EP_CUDA(cudaGetLastError());
  return chebyshev(h, l, b, x);
}

}  // namespace

extern "C" {

int enprop_mg_destroy(enprop_mg* h) {
  if (!h) return ENPROP_OK;
  if (h->ctx) cudaStreamSynchronize(h->ctx->stream);
  for (auto& l : h->lv) free_level(l);
  for (void* q : {(void*)h->lu, (void*)h->luT, (void*)h->piv, (void*)h->r, (void*)h->z, (void*)h->p,
                  (void*)h->q, (void*)h->coef, (void*)h->lanes, (void*)h->act, (void*)h->fin_state})
    if (q) cudaFree(q);
  delete h;
  return ENPROP_OK;
}

int enprop_mg_build(enprop_ctx* c, int s, int rows, const int* row_map, const int* col_entry,
                    const double* values, const enprop_mg_options* opt, enprop_mg** out) {
  ScopedLaunchOpts launch_scope(c);
  if (!c || !out || !row_map || !col_entry || !values) return fail(ENPROP_ERR_INVALID, "build_hierarchy: null argument");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (rows <= 0) return fail(ENPROP_ERR_INVALID, "build_hierarchy: empty matrix");
  enprop_mg_options o{500, 2, 30.0, 1.1, 40};  // MgOptions defaults (multigrid.hpp:14-20)
  if (opt) o = *opt;
  if (o.chebyshev_degree < 1 || o.power_iterations < 0)
    return fail(ENPROP_ERR_INVALID, "build_hierarchy: bad multigrid options");
  auto* h = new (std::nothrow) enprop_mg();
  if (!h) return fail(ENPROP_ERR_OOM, "out of host memory");
  h->ctx = c;
  h->s = s;
  h->opt = o;
  auto bail = [&](int rc) {
    enprop_mg_destroy(h);
    return rc;
  };
  // the fine operator to the host (setup is host-sequential, as in the reference)
  HostCrs a;
  a.rows = a.cols = rows;
  a.rm.resize(rows + 1);
  cudaStream_t st = c->stream;
  if (cudaMemcpyAsync(a.rm.data(), row_map, (rows + 1) * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "build_hierarchy"));
  const int64_t nnz = a.rm[rows];
  a.ce.resize(nnz);
  a.v.resize((size_t)nnz * s);
  if (cudaMemcpyAsync(a.ce.data(), col_entry, nnz * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(a.v.data(), values, (size_t)nnz * s * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "build_hierarchy"));
  int rc = ENPROP_OK;
  // levels (multigrid.hpp:370-389)
  while (a.rows >= o.coarse_row_threshold) {
    std::vector<int> grm, gce, agg;
    connection_graph(a, s, grm, gce);
    const int nc = aggregate_graph(a.rows, grm, gce, agg);
    if (nc >= a.rows) break;
    LevelDev l;
    l.rows = a.rows;
    l.coarse_rows = nc;
    l.nnz = (int64_t)a.ce.size();
    const std::vector<double> diag = diagonal_of(a, s);
    for (double d : diag)
      if (d == 0.0) return bail(fail(ENPROP_ERR_INVALID, "power_lambda_max: zero diagonal entry"));
    // R = P^T (transpose of the one-entry-per-row prolongator, :96-107): row
    // I lists its fine rows ascending, values 1.0
    std::vector<int> rrm(nc + 1, 0), rce(a.rows);
    for (int i = 0; i < a.rows; ++i) ++rrm[agg[i] + 1];
    for (int g = 0; g < nc; ++g) rrm[g + 1] += rrm[g];
    {
      std::vector<int> at(rrm.begin(), rrm.end() - 1);
      for (int i = 0; i < a.rows; ++i) rce[at[agg[i]]++] = i;
    }
    std::vector<double> ones((size_t)a.rows * s, 1.0);
    HostCrs coarse = galerkin_coarse(a, s, agg, nc);
    const size_t vec = (size_t)a.rows * s * sizeof(double);
    if ((rc = upload(&l.rm, a.rm)) || (rc = upload(&l.ce, a.ce)) || (rc = upload(&l.vals, a.v)) ||
        (rc = upload(&l.rrm, rrm)) || (rc = upload(&l.rce, rce)) || (rc = upload(&l.rvals, ones)) ||
        (rc = upload(&l.agg, agg)) || (rc = upload(&l.diag, diag))) {
      free_level(l);
      return bail(rc);
    }
    for (double** vp : {&l.b, &l.x, &l.r, &l.p, &l.tmp})
      if (cudaMalloc(vp, vec) != cudaSuccess) {
        free_level(l);
        return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
      }
    h->lv.push_back(l);
    LevelDev& lv = h->lv.back();  // owned by h from here (bail frees it)
    int pst = 0;
    if ((rc = device_power_lambda_max(h, lv, o.power_iterations, lv.lmax, pst))) return bail(rc);
    if (pst == 2) return bail(fail(ENPROP_ERR_INVALID, "power_lambda_max: iteration collapsed to zero"));
    for (double v : lv.lmax)
      if (v <= 0.0) return bail(fail(ENPROP_ERR_INVALID, "build_hierarchy: non-positive eigenvalue estimate"));
    if ((rc = upload(&lv.cheb, cheb_coeffs(lv.lmax, s, o)))) return bail(rc);
    a = std::move(coarse);
  }
  {  // the coarsest level: dense LU per component on the device (:387-389)
    LevelDev l;
    l.rows = a.rows;
    l.nnz = (int64_t)a.ce.size();
    const size_t vec = (size_t)a.rows * s * sizeof(double);
    if ((rc = upload(&l.rm, a.rm)) || (rc = upload(&l.ce, a.ce)) || (rc = upload(&l.vals, a.v))) return bail(rc);
    for (double** vp : {&l.b, &l.x})
      if (cudaMalloc(vp, vec) != cudaSuccess) return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
    h->lv.push_back(l);
    const int n = a.rows;
    h->coarse_n = n;
    if (lu_solve_smem(n) > 220 * 1024)
      return bail(fail(ENPROP_ERR_INVALID, "build_hierarchy: coarse level too large for the device LU solve"));
    if (lu_solve_smem_optin(s, lu_solve_smem(n)) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "build_hierarchy: coarse solve shared memory"));
    // the dense operator per component, scattered on the device from the
    // coarsest CSR just uploaded (zeros elsewhere, DenseLuSolver's ctor :262-275)
    const size_t dense = (size_t)s * n * n;
    int* singular = nullptr;
    if (cudaMalloc(&h->lu, dense * sizeof(double)) != cudaSuccess)
      return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
    EP_CUDA(cudaMemsetAsync(h->lu, 0, dense * sizeof(double), st));
    k_dense_scatter<<<blocks_for((int64_t)n * s), 256, 0, st>>>(n, s, h->lv.back().rm, h->lv.back().ce,
                                                                  h->lv.back().vals, h->lu);
    c->launches += 1;
    if (cudaMalloc(&h->luT, dense * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&h->piv, (size_t)s * n * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&singular, sizeof(int)) != cudaSuccess)
      return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
    cudaMemsetAsync(singular, 0, sizeof(int), st);
    for (int k0 = 0; k0 < n; k0 += kLuPanel) {  // blocked, with the unblocked algorithm's bits
      const int k1 = std::min(n, k0 + kLuPanel);
      k_lu_factor<<<s * kLuCluster, kLuThreads, 0, st>>>(n, k0, k1, h->lu, h->piv, singular);
      k_lu_swaps<<<dim3((n + 255) / 256, s), 256, 0, st>>>(n, k0, k1, h->lu, h->piv);
      if (k1 < n) {
        k_lu_u12<<<dim3((n - k1 + 127) / 128, s), 128, 0, st>>>(n, k0, k1, h->lu);
        const int tiles = (n - k1 + kLuTile - 1) / kLuTile;
        k_lu_trailing<<<dim3(tiles, tiles, s), 256, 0, st>>>(n, k0, k1, h->lu);
      }
      c->launches += k1 < n ? 4 : 2;
    }
    k_transpose_sq<<<dim3(blocks_for((int64_t)n * n), s), 256, 0, st>>>(n, h->lu, h->luT);
    c->launches += 2;
    int hs = 0;
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaMemcpyAsync(&hs, singular, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    cudaFree(singular);
    if (err != cudaSuccess) return bail(cuda_fail(err, "build_hierarchy: coarse LU"));
    if (hs) return bail(fail(ENPROP_ERR_INVALID, "DenseLuSolver: singular matrix"));
  }
  const int n0 = h->lv[0].rows;
  const size_t vec = (size_t)n0 * s * sizeof(double);
  for (double** vp : {&h->r, &h->z, &h->p, &h->q})
    if (cudaMalloc(vp, vec) != cudaSuccess) return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
  if (cudaMalloc(&h->coef, 2 * kMaxS * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->lanes, (kMaxS + 1) * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->act, kMaxS * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&h->fin_state, sizeof(CgState)) != cudaSuccess)
    return bail(cuda_fail(cudaErrorMemoryAllocation, "build_hierarchy"));
  *out = h;
  return ENPROP_OK;
}

int enprop_mg_describe(enprop_mg* h, int* num_levels, int* rows, int max_levels, double* lambda_max) {
  if (!h) return fail(ENPROP_ERR_INVALID, "null hierarchy");
  const int L = (int)h->lv.size();
  if (num_levels) *num_levels = L;
  for (int k = 0; k < L && k < max_levels; ++k) {
    if (rows) rows[k] = h->lv[k].rows;
    if (lambda_max && k + 1 < L)
      for (int e = 0; e < h->s; ++e) lambda_max[(size_t)k * h->s + e] = h->lv[k].lmax[e];
  }
  return ENPROP_OK;
}

int enprop_mg_vcycle(enprop_mg* h, const double* b, double* x) {
  if (!h || !b || !x) return fail(ENPROP_ERR_INVALID, "vcycle: null argument");
  ScopedLaunchOpts launch_scope(h->ctx);
  return vcycle(h, 0, b, x);
}

}  // extern "C"

namespace {

// serial-order dot (kernels.hpp:62-69) into host lanes[s] (+ coupled sum)
int mg_dot(enprop_mg* h, const double* u, const double* v, std::vector<double>& lanes, double& coupled) {
  const int s = h->s, rows = h->lv[0].rows;
  if (!chain_aligned(u, v)) return fail(ENPROP_ERR_INVALID, "pcg_solve (multigrid): vectors must be 16-byte aligned");
  FinArgs f{};
  f.phase = kPhaseNone;
  f.cg = h->fin_state;
  f.lanes_out = h->lanes;
  EP_CUDA(launch_chain(s, rows, u, v, u == v ? kChainSquare : kChainProduct, f, h->ctx->stream));
  h->ctx->launches += 1;
  std::vector<double> hbuf(s + 1);
  EP_CUDA(cudaMemcpyAsync(hbuf.data(), h->lanes, (s + 1) * sizeof(double), cudaMemcpyDeviceToHost, h->ctx->stream));
  EP_CUDA(cudaStreamSynchronize(h->ctx->stream));
  lanes.assign(hbuf.begin(), hbuf.begin() + s);
  coupled = hbuf[s];
  return ENPROP_OK;
}

int precondition(enprop_mg* h, const double* r, double* z) {
  EP_CUDA(cudaMemsetAsync(z, 0, (size_t)h->lv[0].rows * h->s * sizeof(double), h->ctx->stream));
  return vcycle(h, 0, r, z);  // MgPreconditioner (multigrid.hpp:430-440)
}

}  // namespace

extern "C" {

int enprop_mg_pcg(enprop_mg* h, const double* b, double* x, const enprop_cg_options* opt, int* iterations,
                  int* lane_status, double* history, int* hist_len) {
  if (!h || !b || !x || !opt) return fail(ENPROP_ERR_INVALID, "pcg_solve: null argument");
  ScopedLaunchOpts launch_scope(h->ctx);
  if (opt->dot_mode != ENPROP_DOT_SERIAL)
    return fail(ENPROP_ERR_INVALID, "pcg_solve (multigrid): the reference's serial dot order only");
  const int s = h->s, rows = h->lv[0].rows;
  const bool unc = opt->flavour == ENPROP_CG_UNCOUPLED;
  const int lanes = unc ? s : 1;
  const int maxit = opt->max_iterations;
  cudaStream_t st = h->ctx->stream;
  const size_t vec = (size_t)rows * s * sizeof(double);
  const int64_t n = rows;
  std::vector<std::vector<double>> hist(lanes);
  std::vector<int> its(lanes, 0), status(lanes, 0), active(lanes, 1);
  auto finish = [&](int rc) {
    for (int l = 0; l < lanes; ++l) {
      if (iterations) iterations[l] = its[l];
      if (lane_status) lane_status[l] = status[l];
      if (hist_len) hist_len[l] = (int)hist[l].size();
      if (history)
        for (int it = 0; it <= maxit; ++it)
          history[(size_t)it * lanes + l] = it < (int)hist[l].size() ? hist[l][it] : NAN;
    }
    return rc;
  };
  EP_CUDA(cudaMemsetAsync(x, 0, vec, st));
  std::vector<double> ln;
  double cp = 0.0;
  int rc = mg_dot(h, b, b, ln, cp);  // b_norm = norm2(b)
  if (rc) return rc;
  std::vector<double> bnorm(lanes);
  for (int l = 0; l < lanes; ++l) bnorm[l] = std::sqrt(unc ? ln[l] : cp);
  bool any = false;
  for (int l = 0; l < lanes; ++l) {
    if (bnorm[l] == 0.0) {
      hist[l].push_back(0.0);
      active[l] = 0;
    } else {
      any = true;
    }
  }
  if (!any) return finish(ENPROP_OK);
  EP_CUDA(cudaMemcpyAsync(h->r, b, vec, cudaMemcpyDeviceToDevice, st));
  if ((rc = precondition(h, h->r, h->z))) return rc;
  EP_CUDA(cudaMemcpyAsync(h->p, h->z, vec, cudaMemcpyDeviceToDevice, st));
  if ((rc = mg_dot(h, h->r, h->z, ln, cp))) return rc;
  std::vector<double> rz(lanes);
  for (int l = 0; l < lanes; ++l) rz[l] = unc ? ln[l] : cp;
  std::vector<double> coef(2 * kMaxS, 0.0);
  std::vector<int> act(kMaxS, 0);
  auto upload_coef = [&](const std::vector<double>& a, const std::vector<int>& on) -> int {
    for (int e = 0; e < s; ++e) {
      coef[e] = a[unc ? e : 0];
      act[e] = on[unc ? e : 0];
    }
    EP_CUDA(cudaMemcpyAsync(h->coef, coef.data(), s * sizeof(double), cudaMemcpyHostToDevice, st));
    EP_CUDA(cudaMemcpyAsync(h->act, act.data(), s * sizeof(int), cudaMemcpyHostToDevice, st));
    EP_CUDA(cudaStreamSynchronize(st));  // host buffers are reused next
    return ENPROP_OK;
  };
  int worst = ENPROP_OK;
  for (int it = 0;; ++it) {
    if ((rc = mg_dot(h, h->r, h->r, ln, cp))) return rc;  // norm2(r)
    bool live = false;
    for (int l = 0; l < lanes; ++l) {
      if (!active[l]) continue;
      const double rel = std::sqrt(unc ? ln[l] : cp) / bnorm[l];
      hist[l].push_back(rel);
      if (rel < opt->tol) {
        its[l] = it;
        active[l] = 0;
      } else if (it >= maxit) {
        its[l] = it;
        status[l] = ENPROP_ERR_NO_CONVERGENCE;
        active[l] = 0;
      } else {
        live = true;
      }
    }
    if (!live) break;
    EP_CUDA(spmv_level(h, s, rows, rows, h->lv[0].rm, h->lv[0].ce, h->lv[0].vals, h->p, h->q));
    if ((rc = mg_dot(h, h->p, h->q, ln, cp))) return rc;
    std::vector<double> alpha(lanes, 0.0), malpha(lanes, 0.0);
    for (int l = 0; l < lanes; ++l) {
      if (!active[l]) continue;
      const double pq = unc ? ln[l] : cp;
      if (pq <= 0.0) {
        status[l] = ENPROP_ERR_INDEFINITE;
        its[l] = it;
        active[l] = 0;
        continue;
      }
      alpha[l] = rz[l] / pq;
      malpha[l] = -alpha[l];
    }
    if ((rc = upload_coef(alpha, active))) return rc;  // x = alpha*p + 1.0*x
    EP_MG_DISPATCH(s, k_axpy_masked, blocks_for(n * s), 256, 0, st, n, h->coef, h->act, h->p, x);
    if ((rc = upload_coef(malpha, active))) return rc;  // r = -alpha*q + 1.0*r
    EP_MG_DISPATCH(s, k_axpy_masked, blocks_for(n * s), 256, 0, st, n, h->coef, h->act, h->q, h->r);
    h->ctx->launches += 2;
    if ((rc = precondition(h, h->r, h->z))) return rc;
    if ((rc = mg_dot(h, h->r, h->z, ln, cp))) return rc;
    std::vector<double> beta(lanes, 0.0);
    for (int l = 0; l < lanes; ++l) {
      if (!active[l]) continue;
      const double rz_next = unc ? ln[l] : cp;
      beta[l] = rz_next / rz[l];
      rz[l] = rz_next;
    }
    if ((rc = upload_coef(beta, active))) return rc;  // p = 1.0*z + beta*p
    EP_MG_DISPATCH(s, k_direction_masked, blocks_for(n * s), 256, 0, st, n, h->coef, h->act, h->z, h->p);
    h->ctx->launches += 1;
    EP_CUDA(cudaGetLastError());
  }
  EP_CUDA(cudaStreamSynchronize(st));
  for (int l = 0; l < lanes; ++l) worst = std::max(worst, status[l]);
  finish(ENPROP_OK);
  if (worst == ENPROP_ERR_NO_CONVERGENCE)
    return fail(ENPROP_ERR_NO_CONVERGENCE, "pcg_solve: no convergence within " + std::to_string(maxit) + " iterations");
  if (worst == ENPROP_ERR_INDEFINITE)
    return fail(ENPROP_ERR_INDEFINITE, "pcg_solve: operator not positive definite (p'Ap <= 0)");
  return ENPROP_OK;
}

}  // extern "C"
