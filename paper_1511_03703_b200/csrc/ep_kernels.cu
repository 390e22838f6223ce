// enprop_b200 kernels for sm_100a.
//
// Ensemble layout (reference ensemble.hpp:105-106): the s sample values of each
// stored entry and of each vector row are contiguous, so one nonzero's s
// values are one coalesced 8s-byte chunk.  Lanes of the SIMT mapping carry
// samples: a row is handled by TPR = s/V threads, each owning V consecutive
// samples and loading them with one 16-byte vector load.
//
// Parity: per-sample arithmetic reproduces the reference's sequence of IEEE
// operations exactly (no FMA, same order), so assembly, Dirichlet, SpMV and
// axpby are bitwise equal to proj/include/enprop/{fem,kernels}.hpp.
#include <cstdio>

#include "ep_common.cuh"
#include "ep_kernels.h"
#include "ep_fin.cuh"

namespace ep {

// =============================================================================
// Node graph (proj/src/mesh.cpp:13-55) built on the device in closed form.
// Row (i,j,k) of the x-fastest numbering has C(i)C(j)C(k) entries, C(t) = 2 at
// the two ends of an axis and 3 inside; its first entry is
//   P(k) W^2 + C(k) (P(j) W + C(j) P(i)),  P(t) = sum_{t'<t} C(t'), W = 3N-2,
// and its columns are listed kk -> jj -> ii ascending, as the reference does.
// =============================================================================
__device__ __forceinline__ int axis_count(int t, int N) { return 1 + (t > 0) + (t < N - 1); }
__device__ __forceinline__ int axis_prefix(int t) { return t == 0 ? 0 : 2 + 3 * (t - 1); }

__global__ void k_build_graph(int n, int* __restrict__ row_map, int* __restrict__ col_entry) {
  const int N = n + 1;
  const int rows = N * N * N;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int i = row % N, j = (row / N) % N, k = row / (N * N);
  const int W = 3 * N - 2;
  const int ci = axis_count(i, N), cj = axis_count(j, N), ck = axis_count(k, N);
  const int start = axis_prefix(k) * W * W + ck * (axis_prefix(j) * W + cj * axis_prefix(i));
  if (row == 0) row_map[0] = 0;
  row_map[row + 1] = start + ci * cj * ck;
  int at = start;
  const int ilo = i > 0 ? i - 1 : 0, ihi = i < N - 1 ? i + 1 : N - 1;
  const int jlo = j > 0 ? j - 1 : 0, jhi = j < N - 1 ? j + 1 : N - 1;
  const int klo = k > 0 ? k - 1 : 0, khi = k < N - 1 ? k + 1 : N - 1;
  for (int kk = klo; kk <= khi; ++kk)
    for (int jj = jlo; jj <= jhi; ++jj)
      for (int ii = ilo; ii <= ihi; ++ii) col_entry[at++] = ii + N * (jj + N * kk);
}

__global__ void k_build_graph_range(int n, int row_begin, int nrows, int col_shift,
                                    int* __restrict__ row_map, int* __restrict__ col_entry) {
  const int N = n + 1;
  const int W = 3 * N - 2;
  const int lrow = blockIdx.x * blockDim.x + threadIdx.x;
  if (lrow >= nrows) return;
  auto start_of = [&](int row) {
    const int i = row % N, j = (row / N) % N, k = row / (N * N);
    return axis_prefix(k) * W * W +
           axis_count(k, N) * (axis_prefix(j) * W + axis_count(j, N) * axis_prefix(i));
  };
  const int row = row_begin + lrow;
  const int i = row % N, j = (row / N) % N, k = row / (N * N);
  const int base = start_of(row_begin);
  const int start = start_of(row) - base;
  if (lrow == 0) row_map[0] = 0;
  row_map[lrow + 1] = start + axis_count(i, N) * axis_count(j, N) * axis_count(k, N);
  int at = start;
  const int ilo = i > 0 ? i - 1 : 0, ihi = i < N - 1 ? i + 1 : N - 1;
  const int jlo = j > 0 ? j - 1 : 0, jhi = j < N - 1 ? j + 1 : N - 1;
  const int klo = k > 0 ? k - 1 : 0, khi = k < N - 1 ? k + 1 : N - 1;
  for (int kk = klo; kk <= khi; ++kk)
    for (int jj = jlo; jj <= jhi; ++jj)
      for (int ii = ilo; ii <= ihi; ++ii) col_entry[at++] = ii + N * (jj + N * kk) - col_shift;
}

cudaError_t launch_build_graph_range(int n, int row_begin, int rows, int col_shift, int* row_map,
                                     int* col_entry, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  k_build_graph_range<<<(rows + 255) / 256, 256, 0, st>>>(n, row_begin, rows, col_shift, row_map, col_entry);
  return cudaGetLastError();
}

cudaError_t launch_build_graph(int n, int* row_map, int* col_entry, cudaStream_t st) {
  const int N = n + 1;
  const int rows = N * N * N;
  k_build_graph<<<(rows + 255) / 256, 256, 0, st>>>(n, row_map, col_entry);
  return cudaGetLastError();
}

// =============================================================================
// SpMV building block (kernels.hpp:15-26): one row, V samples of this thread.
// sum = 0; sum += a_k * x_col_k in entry order — the reference's per-sample
// sequence.  Entries are processed in predicated batches of U so the column,
// value and gather loads of a batch are all in flight together; invalid batch
// slots are skipped (never "+0.0") so the order and bits stay the reference's.
// With kCg the gathered operand is p_new = r + beta*p_old formed on the fly
// (first iteration: p_new = r), which removes a separate direction pass.
// =============================================================================
template <int S>
struct SpmvShape {  // vector width per thread
  static constexpr int V = (S == 1) ? 1 : 2;
  static constexpr int TPR = S / V;
  static constexpr int U = 4;  // entries per predicated batch
};

// kSym: values are the symmetric (diagonal + upper) storage and entry k's
// value lives at vpos[k] (its own slot for col >= row, the transposed slot in
// row col's upper part otherwise); the per-row summation order is unchanged.
template <int S, int V, int U, bool kCg, bool kPipe = false, bool kSym = false>
__device__ __forceinline__ VecD<V> row_product(int row, const int* __restrict__ row_map,
                                               const int* __restrict__ col_entry,
                                               const double* __restrict__ values,
                                               const double* __restrict__ x_or_r,
                                               const double* __restrict__ p_old, bool first,
                                               const VecD<V>& beta, int lane0,
                                               const int* __restrict__ vpos = nullptr) {
  const int rs = __ldg(row_map + row), re = __ldg(row_map + row + 1);
  VecD<V> sum;
#pragma unroll
  for (int j = 0; j < V; ++j) sum.v[j] = 0.0;
  // kPipe: column indices run one batch ahead of the gathers (software
  // pipelining). Measured slower on B200 (6235 -> 4968 GB/s at 128^3), so off
  // by default; kept for tuning (ENPROP_OPT_SPMV_PIPELINE).
  int cn[U];
  if constexpr (kPipe) {
#pragma unroll
    for (int u = 0; u < U; ++u) cn[u] = (rs + u < re) ? ld_stream_i32(col_entry + rs + u) : 0;
  }
  for (int kb = rs; kb < re; kb += U) {
    int c[U];
    VecD<V> av[U], xv[U], pv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = kPipe ? cn[u] : ((kb + u < re) ? ld_stream_i32(col_entry + kb + u) : 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kb + u < re) {
        const size_t vi = kSym ? (size_t)ld_stream_i32(vpos + kb + u) : (size_t)(kb + u);
        av[u] = ld_stream<V>(values + vi * S + lane0);
        xv[u] = ld_vec<V>(x_or_r + (size_t)c[u] * S + lane0);
        if (kCg && !first) pv[u] = ld_vec<V>(p_old + (size_t)c[u] * S + lane0);
      }
    }
    if constexpr (kPipe) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        cn[u] = (kb + U + u < re) ? ld_stream_i32(col_entry + kb + U + u) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kb + u < re) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          double xo = xv[u].v[j];
          if (kCg && !first) xo = EP_DADD(xo, EP_DMUL(beta.v[j], pv[u].v[j]));
          sum.v[j] = EP_DADD(sum.v[j], EP_DMUL(av[u].v[j], xo));
        }
      }
    }
  }
  return sum;
}

template <int S, bool kPipe>
__global__ void __launch_bounds__(256) k_spmv(int rows, const int* __restrict__ row_map,
                                              const int* __restrict__ col_entry,
                                              const double* __restrict__ values,
                                              const double* __restrict__ x,
                                              double* __restrict__ z) {
  using Sh = SpmvShape<S>;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt / Sh::TPR;
  const int lane0 = (gt - row * Sh::TPR) * Sh::V;
  if (row >= rows) return;
  VecD<Sh::V> beta;
  const VecD<Sh::V> sum = row_product<S, Sh::V, Sh::U, false, kPipe>(row, row_map, col_entry,
                                                                      values, x, nullptr, true,
                                                                      beta, lane0);
  st_vec<Sh::V>(z + (size_t)row * S + lane0, sum);
}

template <int S>
static cudaError_t spmv_s(int rows, const int* row_map, const int* col_entry,
                          const double* values, const double* x, double* z, bool pipe,
                          cudaStream_t st) {
  using Sh = SpmvShape<S>;
  const int64_t threads = (int64_t)rows * Sh::TPR;
  if (threads == 0) return cudaSuccess;
  const int grid = (int)((threads + 255) / 256);
  if (pipe) k_spmv<S, true><<<grid, 256, 0, st>>>(rows, row_map, col_entry, values, x, z);
  else k_spmv<S, false><<<grid, 256, 0, st>>>(rows, row_map, col_entry, values, x, z);
  return cudaGetLastError();
}

cudaError_t launch_spmv(int s, int rows, const int* row_map, const int* col_entry,
                        const double* values, const double* x, double* z, bool pipe,
                        cudaStream_t st) {
  EP_DISPATCH_S(s, spmv_s, rows, row_map, col_entry, values, x, z, pipe, st);
}

// =============================================================================
// axpby (kernels.hpp:78-85): y = alpha*x + beta*y, per lane or scalar coefs.
// =============================================================================
template <int S>
__global__ void __launch_bounds__(256) k_axpby(int64_t n, const double* __restrict__ alpha,
                                               const double* __restrict__ beta,
                                               const double* __restrict__ x,
                                               double* __restrict__ y) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n * S) return;
  const int e = (int)(g % S);
  y[g] = EP_DADD(EP_DMUL(alpha[e], x[g]), EP_DMUL(beta[e], y[g]));
}

template <int S>
static cudaError_t axpby_s(int64_t n, const double* alpha, const double* beta, const double* x,
                           double* y, cudaStream_t st) {
  const int64_t t = n * S;
  if (t == 0) return cudaSuccess;
  k_axpby<S><<<(int)((t + 255) / 256), 256, 0, st>>>(n, alpha, beta, x, y);
  return cudaGetLastError();
}

cudaError_t launch_axpby(int s, int64_t n, int /*per_lane*/, const double* alpha,
                         const double* beta, const double* x, double* y, cudaStream_t st) {
  // alpha/beta are device arrays of s coefficients (replicated when scalar)
  EP_DISPATCH_S(s, axpby_s, n, alpha, beta, x, y, st);
}

// =============================================================================
// Canonical reduction (restated by oracle/enprop_oracle.c
// or_dot_lanes).  Rows are cut into segments of seg_rows (a mesh z-plane) and
// each segment into tiles of kTileRows = 16 rows aligned at the segment start.
// Per sample:  tile sum  = stride-halving tree v[i] += v[i+h], h = 8,4,2,1
//                          over the tile's products (+0.0 past the tile end);
//              segment   = 0.0 + tile_0 + tile_1 + ...      (sequential)
//              total     = 0.0 + seg_0 + seg_1 + ...        (sequential)
// A block owns TPC whole tiles.  The finalize is fused into the producing
// kernel: after writing its tile partials, a block bumps its segments' arrival
// counters; the block that completes a segment forms the segment sum, and the
// block that completes the last segment forms the total and runs the CG scalar
// phase.  Counters reset themselves, so no launch or memset sits between.
// =============================================================================
// Block shape: NT threads, TPR threads per row, RPC row slots per pass, P
// passes per block (a thread owns P rows; their loads are issued together).
template <int S, int P = 1, int NT_ = 256>
struct TileShape {
  static constexpr int V = SpmvShape<S>::V;
  static constexpr int TPR = S / V;                // threads per row
  static constexpr int NT = NT_;                   // threads per block
  static constexpr int RPC = NT / TPR;             // row slots per pass
  static constexpr int ROWS = RPC * P;             // row slots per block
  static constexpr int TPC = ROWS / kTileRows;     // tiles per block
  static_assert(ROWS % kTileRows == 0, "a block must cover whole tiles");
};


// Row of block slot `slot` in canonical tiling (-1: none).
template <int S, int P, int NT = 256>
__device__ __forceinline__ int tile_row(const TileMap& tm, int slot) {
  using Sh = TileShape<S, P, NT>;
  const int tile = blockIdx.x * Sh::TPC + slot / kTileRows;
  if (tile >= tm.num_tiles()) return -1;
  int r0, nr;
  tm.tile(tile, r0, nr);
  const int ri = slot % kTileRows;
  return ri < nr ? r0 + ri : -1;
}

// Tile trees: every thread has stored its rows' products in sprod[slot][S];
// after one barrier, thread (tile, sample) folds the tile's 16 rows in
// registers in the canonical order (v[i] += v[i+h], h = 8,4,2,1; rows past the
// tile end hold +0.0) and writes the tile partial. The dot is closed by
// k_fin_segments, so blocks retire right after this (no global round trip).
template <int S, int P, int NT = 256>
__device__ __forceinline__ void tiles_finish(const TileMap& tm, const double* sprod, const FinArgs& f) {
  using Sh = TileShape<S, P, NT>;
  __syncthreads();
  for (int idx = threadIdx.x; idx < Sh::TPC * S; idx += Sh::NT) {
    const int lt = idx / S, e = idx - lt * S;
    const int tile = blockIdx.x * Sh::TPC + lt;
    if (tile >= tm.num_tiles()) continue;
    int r0, nr;
    tm.tile(tile, r0, nr);
    if (nr <= 0) continue;
    double v[kTileRows];
#pragma unroll
    for (int i = 0; i < kTileRows; ++i) v[i] = sprod[(lt * kTileRows + i) * S + e];
#pragma unroll
    for (int h = kTileRows / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int i = 0; i < h; ++i) v[i] = EP_DADD(v[i], v[i + h]);
    f.partials[(size_t)tile * S + e] = v[0];
  }
}

constexpr int kStreamPasses = 4;  // rows per thread in the streaming (dot/update) kernels

template <int S>
__global__ void __launch_bounds__(256) k_dot_tiles(const TileMap tm, const double* __restrict__ u,
                                                   const double* __restrict__ v, const FinArgs f) {
  EP_PDL_ENTRY();
  constexpr int P = kStreamPasses;
  using Sh = TileShape<S, P>;
  constexpr int V = Sh::V;
  __shared__ double sprod[Sh::ROWS * S];
  const int lane0 = (threadIdx.x % Sh::TPR) * V;
  VecD<V> a[P], b[P];
  int row[P];
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    row[ps] = tile_row<S, P>(tm, ps * Sh::RPC + threadIdx.x / Sh::TPR);
    if (row[ps] >= 0) {
      a[ps] = ld_vec<V>(u + (size_t)row[ps] * S + lane0);
      b[ps] = ld_vec<V>(v + (size_t)row[ps] * S + lane0);
    }
  }
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    const int slot = ps * Sh::RPC + threadIdx.x / Sh::TPR;
#pragma unroll
    for (int j = 0; j < V; ++j)
      sprod[slot * S + lane0 + j] = row[ps] >= 0 ? EP_DMUL(a[ps].v[j], b[ps].v[j]) : 0.0;
  }
  tiles_finish<S, P>(tm, sprod, f);
}

template <int S>
static cudaError_t dot_tiles_s(const TileMap& tm, const double* u, const double* v,
                               const FinArgs& f, cudaStream_t st) {
  using Sh = TileShape<S, kStreamPasses>;
  const int blocks = (tm.num_tiles() + Sh::TPC - 1) / Sh::TPC;
  if (blocks == 0) return cudaSuccess;
  launch_kk(16, k_dot_tiles<S>, dim3(blocks), dim3(Sh::NT), 0, st, tm, u, v, f);
  return cudaGetLastError();
}

cudaError_t launch_dot_tiles(int s, const TileMap& tm, const double* u, const double* v,
                             const FinArgs& f, cudaStream_t st) {
  EP_DISPATCH_S(s, dot_tiles_s, tm, u, v, f, st);
}

// Canonical finalize, one CTA per segment (ep_fin.cuh fin_segment_fold /
// fin_total_phase, shared with the staged SpMV's fused tail).
template <int S>
__global__ void __launch_bounds__(kFinThreads) k_fin_segments(const TileMap tm, const FinArgs f) {
  EP_PDL_ENTRY();
  if ((f.phase == kPhasePQ || f.phase == kPhaseRR) && f.cg->done) return;
  __shared__ double sblk[FinShape<S>::CHUNK * S];
  __shared__ double stot[FinShape<S>::CHUNK2 * S];
  __shared__ double lanes[S];
  __shared__ int s_final;
  fin_segment_fold<S>(tm, f, blockIdx.x, sblk);
  if (f.seg_only) return;
  fin_total_phase<S>(tm, f, stot, lanes, &s_final);
}

template <int S>
static cudaError_t fin_segments_s(const TileMap& tm, const FinArgs& f, cudaStream_t st) {
  if (tm.num_segs == 0) return cudaSuccess;
  launch_kk(4, k_fin_segments<S>, dim3(tm.num_segs), dim3(kFinThreads), 0, st, tm, f);
  return cudaGetLastError();
}

cudaError_t launch_fin_segments(int s, const TileMap& tm, const FinArgs& f, cudaStream_t st) {
  EP_DISPATCH_S(s, fin_segments_s, tm, f, st);
}

// Multi-GPU canonical total: lanes[e] = 0.0 + seg_0 + seg_1 + ... over the
// global planes in order, read from the all-gathered per-rank segment sums
// (gathered[plane_pos[k]][e]); then the CG scalar phase. Every rank runs it on
// identical data, so all ranks take identical decisions.
template <int S>
__global__ void __launch_bounds__(256) k_fin_gathered(int planes, const double* __restrict__ gathered,
                                                      const int* __restrict__ plane_pos, int phase,
                                                      CgState* cg, double* hist, double* lanes_out) {
  EP_PDL_ENTRY();
  if ((phase == kPhasePQ || phase == kPhaseRR) && cg->done) return;
  constexpr int kChunk = 64;
  __shared__ double sch[kChunk * S];
  __shared__ double lanes[S];
  double tot = 0.0;
  for (int k0 = 0; k0 < planes; k0 += kChunk) {
    const int cnt = min(kChunk, planes - k0);
    for (int idx = threadIdx.x; idx < cnt * S; idx += blockDim.x) {
      const int k = idx / S, e = idx - k * S;
      sch[idx] = gathered[(size_t)plane_pos[k0 + k] * S + e];
    }
    __syncthreads();
    if (threadIdx.x < S)
      for (int k = 0; k < cnt; ++k) tot = EP_DADD(tot, sch[k * S + threadIdx.x]);
    __syncthreads();
  }
  if (threadIdx.x < S) lanes[threadIdx.x] = tot;
  __syncthreads();
  if (threadIdx.x < 32) cg_phase<S>(phase, lanes, cg, hist, lanes_out);
}

template <int S>
static cudaError_t fin_gathered_s(int planes, const double* gathered, const int* plane_pos,
                                  int phase, CgState* cg, double* hist, double* lanes_out,
                                  cudaStream_t st) {
  launch_kk(4, k_fin_gathered<S>, dim3(1), dim3(256), 0, st, planes, gathered, plane_pos, phase, cg, hist, lanes_out);
  return cudaGetLastError();
}

cudaError_t launch_fin_gathered(int s, int planes, const double* gathered, const int* plane_pos,
                                int phase, CgState* cg, double* hist, double* lanes_out,
                                cudaStream_t st) {
  EP_DISPATCH_S(s, fin_gathered_s, planes, gathered, plane_pos, phase, cg, hist, lanes_out, st);
}

// Serial finalize: the reference's own order (kernels.hpp:66-67), one chain
// per sample: acc = 0; acc += u[row]*v[row] for row = 0, 1, ...  The chain is
// latency-bound (one dependent DADD per row, ~8 cycles on B200), so the design
// keeps the chain's operands in registers (enprop_dot's path for operands that
// are not 16-byte aligned; the CG loop uses k_chain): one warp per sample; in a chunk of
// 32*K rows lane j holds the products of rows [jK, jK+K) and the running sum
// walks lane 0 -> lane 31 by shuffles, while the next chunk's loads are in
// flight.  A block holds the warps of LG = min(s, 4) samples (one 32-byte
// sector per row, shared through L1).  The last block to finish (acq_rel
// counter) runs the scalar phase on all s lanes.
constexpr int kSerialK = 16;  // rows per lane per chunk

template <int S>
struct SerialShape {
  static constexpr int LG = S < 4 ? S : 4;  // samples (warps) per block
  static constexpr int GROUPS = S / LG;
  static constexpr int CHUNK = 32 * kSerialK;
};

template <int S>
__global__ void __launch_bounds__(32 * SerialShape<S>::LG) k_fin_serial(
    int rows, const double* __restrict__ u, const double* __restrict__ v, const FinArgs f) {
  EP_PDL_ENTRY();
  using Sh = SerialShape<S>;
  constexpr int K = kSerialK;
  if ((f.phase == kPhasePQ || f.phase == kPhaseRR) && f.cg->done) return;
  __shared__ double lanes[S];
  __shared__ int s_final;
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * Sh::LG + (threadIdx.x >> 5);  // this warp's sample
  const int nchunks = (rows + Sh::CHUNK - 1) / Sh::CHUNK;
  double ua[K], va[K], cur[K];
  auto load = [&](int c) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int row = c * Sh::CHUNK + lane * K + k;
      if (row < rows) {
        ua[k] = __ldg(u + (size_t)row * S + e);
        va[k] = __ldg(v + (size_t)row * S + e);
      }
    }
  };
  double acc = 0.0;
  if (nchunks > 0) {
    load(0);
#pragma unroll
    for (int k = 0; k < K; ++k) cur[k] = EP_DMUL(ua[k], va[k]);
  }
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) load(c + 1);  // in flight during the chain
    const int base = c * Sh::CHUNK;
    if (base + Sh::CHUNK <= rows) {
      // full chunk: every lane runs the same unpredicated chain on its own
      // registers in lockstep (no divergence); the shuffle keeps lane j's
      // result, which is the running sum through row base + (j+1)K - 1
      for (int j = 0; j < 32; ++j) {
        double t = acc;
#pragma unroll
        for (int k = 0; k < K; ++k) t = EP_DADD(t, cur[k]);
        acc = __shfl_sync(0xffffffffu, t, j);
      }
    } else {
      for (int j = 0; j < 32; ++j) {
        double t = acc;
        const int nv = rows - (base + j * K);  // rows of lane j in this chunk
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (k < nv) t = EP_DADD(t, cur[k]);
        acc = __shfl_sync(0xffffffffu, t, j);
      }
    }
    if (c + 1 < nchunks) {
#pragma unroll
      for (int k = 0; k < K; ++k) cur[k] = EP_DMUL(ua[k], va[k]);
    }
  }
  if (lane == 0) {
    f.seg_sums[e] = acc;
    // every writing warp fences its own store: thread 0's release below only
    // covers its own warp's stores, and the last block reads all of them
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) s_final = (atomic_add_acq_rel_gpu(f.seg_done, 1) == Sh::GROUPS - 1);
  __syncthreads();
  if (s_final) {
    if (threadIdx.x < S) lanes[threadIdx.x] = __ldcg(f.seg_sums + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) *f.seg_done = 0;
    if (threadIdx.x < 32) cg_phase<S>(f.phase, lanes, f.cg, f.hist, f.lanes_out);
  }
}

template <int S>
static cudaError_t fin_serial_s(int rows, const double* u, const double* v, const FinArgs& f,
                                cudaStream_t st) {
  using Sh = SerialShape<S>;
  launch_kk(4, k_fin_serial<S>, dim3(Sh::GROUPS), dim3(32 * Sh::LG), 0, st, rows, u, v, f);
  return cudaGetLastError();
}

cudaError_t launch_fin_serial(int s, int rows, const double* u, const double* v, const FinArgs& f,
                              cudaStream_t st) {
  EP_DISPATCH_S(s, fin_serial_s, rows, u, v, f, st);
}

// =============================================================================
// CG vector kernels.  Flat row mapping: TPR threads per row, one row per slot,
// P slots per thread, so every row of the grid is in flight at once.  With
// kTiles the slots are the block's canonical tiles and the fused finalize
// closes the dot; without (serial order) rows are contiguous and the chain
// kernel (ep_chain.cu) forms the dot.  All kernels early-exit once the solve is done,
// so the host may enqueue ahead of its convergence check.
// =============================================================================
template <int S, int P, bool kTiles, int NT = 256>
__device__ __forceinline__ int cg_row(const TileMap& tm, int slot) {
  if constexpr (kTiles) {
    return tile_row<S, P, NT>(tm, slot);
  } else {
    const int row = blockIdx.x * TileShape<S, P, NT>::ROWS + slot;
    return row < tm.rows ? row : -1;
  }
}

// q = A p_new.  kFusedDir: p_new = (it == 0 ? r : r + beta*p_old) is formed on
// the fly from gathers of r and p_old and written for the block's own rows
// (saves the direction pass). Otherwise p_new was written by k_cg_direction
// and is gathered directly (one gather per entry).  Both give the reference's
// p = 1.0*z + beta*p (pcg.hpp:101) bit for bit.
template <int S, bool kTiles, bool kFusedDir, bool kSym = false>
__global__ void __launch_bounds__(256, 4) k_cg_spmv(
    const TileMap tm, const int* __restrict__ row_map, const int* __restrict__ col_entry,
    const double* __restrict__ values, const double* __restrict__ r,
    const double* __restrict__ p_old, double* __restrict__ p_new, double* __restrict__ q,
    double* __restrict__ x, const double* __restrict__ p_gather, const int* __restrict__ vpos,
    const FinArgs f) {
  EP_PDL_ENTRY();
  using Sh = TileShape<S, 1>;
  constexpr int V = Sh::V;
  const CgState* cg = f.cg;
  if (cg->done) return;
  __shared__ double sprod[kTiles ? Sh::ROWS * S : 1];
  const int slot = threadIdx.x / Sh::TPR;
  const int lane0 = (threadIdx.x % Sh::TPR) * V;
  const bool first = cg->it == 0;
  VecD<V> beta;
#pragma unroll
  for (int j = 0; j < V; ++j) beta.v[j] = cg->beta[lane0 + j];
  const int row = cg_row<S, 1, kTiles>(tm, slot);
  VecD<V> pr;
  if (row >= 0) {
    VecD<V> sum, pn;
    if constexpr (kFusedDir) {
      sum = row_product<S, V, SpmvShape<S>::U, true>(row, row_map, col_entry, values, r, p_old,
                                                     first, beta, lane0);
      pn = ld_vec<V>(r + (size_t)row * S + lane0);
      if (!first) {
        const VecD<V> po = ld_vec<V>(p_old + (size_t)row * S + lane0);
        VecD<V> xv = ld_vec<V>(x + (size_t)row * S + lane0);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          pn.v[j] = EP_DADD(pn.v[j], EP_DMUL(beta.v[j], po.v[j]));
          if (cg->pending[lane0 + j]) xv.v[j] = EP_DADD(EP_DMUL(cg->alpha[lane0 + j], po.v[j]), xv.v[j]);
        }
        st_vec<V>(x + (size_t)row * S + lane0, xv);
      }
      st_vec<V>(p_new + (size_t)row * S + lane0, pn);
    } else {
      sum = row_product<S, V, SpmvShape<S>::U, false, false, kSym>(
          row, row_map, col_entry, values, p_gather, nullptr, true, beta, lane0, vpos);
      pn = ld_vec<V>(p_new + (size_t)row * S + lane0);
    }
    st_vec<V>(q + (size_t)row * S + lane0, sum);
#pragma unroll
    for (int j = 0; j < V; ++j) pr.v[j] = EP_DMUL(pn.v[j], sum.v[j]);
    if (!kTiles && f.prod) st_vec<V>(f.prod + (size_t)row * S + lane0, pr);
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) pr.v[j] = 0.0;
  }
  if constexpr (kTiles) {
#pragma unroll
    for (int j = 0; j < V; ++j) sprod[slot * S + lane0 + j] = pr.v[j];
    tiles_finish<S, 1>(tm, sprod, f);
  }
}

// -----------------------------------------------------------------------------
// Warp-per-tile CG SpMV (split-direction schedule, the default): q = A p and
// the canonical p.q tile partials with no shared memory and no barrier.
//
// A warp owns TILES whole tiles (or, in serial order, 16 contiguous rows) and
// walks them in PASSES passes of R = 32/TPR rows; thread (g, sub) handles row
// g of each pass, lanes [sub*V, sub*V+V). Tile row r = ps*R + g, so the tree
// levels h >= R of the canonical tile fold (v[r] += v[r+h], h = 8,4,2,1) pair
// rows held by the same thread (register adds) and the levels h < R pair
// threads h*TPR apart (shuffles).
//
// Row products load the row's column indices (and symmetric slots)
// cooperatively -- each of the row's TPR threads loads E of the window's
// W = TPR*E entries -- and broadcast them by shuffle, so each batch of U
// gathers waits on one memory latency instead of two.
// -----------------------------------------------------------------------------
// ENPROP_OPT_SPMV_VARIANT of the calling context (-1 auto, see SpmvVariant)
int spmv_variant() {
  const int v = launch_opts().spmv_variant;
  return (v >= 0 && v <= 6) ? v : -1;
}

// Vector kernels of the CG loop run 128-thread blocks capped at 48 registers
// (kVecNT): small enough to be co-resident with a staged-SpMV CTA of another
// sample group (which leaves ~6 K registers and ~17 KB of shared memory per
// SM), so concurrent groups overlap their HBM-bound passes with the SpMV.
constexpr int kVecNT = 128;

// block size of the CG vector kernels (ENPROP_VEC_NT env: 128 default, or 256)
int vec_nt() {
  static const int nt = env_int("ENPROP_VEC_NT", kVecNT) == 256 ? 256 : kVecNT;
  return nt;
}

template <int S>
struct WarpTile {
  static constexpr int V = SpmvShape<S>::V;
  static constexpr int TPR = S / V;                                  // threads per row
  static constexpr int R = 32 / TPR;                                 // rows per warp pass
  static constexpr int PASSES = R >= kTileRows ? 1 : kTileRows / R;  // passes per tile
  static constexpr int TILES = R >= kTileRows ? R / kTileRows : 1;   // tiles per warp
  static constexpr int E = TPR >= 4 ? 32 / TPR : 0;                  // index loads per thread
  static constexpr int W = TPR * E;                                  // window (entries)
};

// Index window of one row: its CRS range and the first W column indices (and
// symmetric slots), E per thread, loaded by the row's TPR threads together.
template <int S>
struct RowIdx {
  static constexpr int E = WarpTile<S>::E > 0 ? WarpTile<S>::E : 1;
  int rs, n;
  int mc[E], mv[E];
};

template <int S, bool kSym>
__device__ __forceinline__ void row_index(int row, const int* __restrict__ row_map,
                                          const int* __restrict__ col_entry,
                                          const int* __restrict__ vpos, int sub, uint64_t pol,
                                          RowIdx<S>& ix) {
  using Sh = WarpTile<S>;
  ix.rs = 0;
  ix.n = 0;
  if (row >= 0) {
    ix.rs = __ldg(row_map + row);
    ix.n = __ldg(row_map + row + 1) - ix.rs;
  }
  if constexpr (Sh::E > 0) {
#pragma unroll
    for (int i = 0; i < Sh::E; ++i) {
      const int k = i * Sh::TPR + sub;
      ix.mc[i] = k < ix.n ? ld_stream_i32_hint(col_entry + ix.rs + k, pol) : 0;
      if constexpr (kSym) ix.mv[i] = k < ix.n ? ld_stream_i32_hint(vpos + ix.rs + k, pol) : 0;
    }
  }
}

// Row product from a loaded index window: batches of U entries, each batch's
// value and vector gathers issued together (the indices come by shuffle), so a
// batch waits on one memory latency. Every lane of the warp must call this
// (warp-uniform trip counts via __reduce_max_sync).
// L2 policy: all streams are read with an explicit cache policy -- the default
// for ld.global.nc.L1::no_allocate let the upper slots fall out of L2 before
// their transposed re-read (1.68 vs 1.29 GB DRAM per SpMV at 64^3, s = 32).
template <int S, bool kSym, int U, bool kPadZero>
__device__ __forceinline__ VecD<SpmvShape<S>::V> row_compute(
    int row, const RowIdx<S>& ix, const int* __restrict__ row_map,
    const int* __restrict__ col_entry, const double* __restrict__ values,
    const double* __restrict__ x, const int* __restrict__ vpos, int sub, uint64_t pol) {
  using Sh = WarpTile<S>;
  constexpr int V = Sh::V, TPR = Sh::TPR, E = Sh::E, W = Sh::W;
  const int lane0 = sub * V;
  VecD<V> sum;
#pragma unroll
  for (int j = 0; j < V; ++j) sum.v[j] = 0.0;
  if constexpr (E == 0) {  // narrow rows (TPR < 4): plain per-thread loop
    if (row >= 0) {
      VecD<V> beta;
      sum = row_product<S, V, 4, false, false, kSym>(row, row_map, col_entry, values, x, nullptr,
                                                     true, beta, lane0, vpos);
    }
    return sum;
  } else {
    const int rs = ix.rs, n = ix.n;
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    const int gbase = (threadIdx.x & 31) - sub;  // first lane of this row's group
    for (int w0 = 0; w0 < nmax; w0 += W) {
      int mc[E], mv[E];
#pragma unroll
      for (int i = 0; i < E; ++i) {
        if (w0 == 0) {
          mc[i] = ix.mc[i];
          mv[i] = ix.mv[i];
        } else {  // rows longer than one window (general graphs)
          const int k = w0 + i * TPR + sub;
          mc[i] = k < n ? ld_stream_i32_hint(col_entry + rs + k, pol) : 0;
          if constexpr (kSym) mv[i] = k < n ? ld_stream_i32_hint(vpos + rs + k, pol) : 0;
        }
      }
#pragma unroll
      for (int kb = 0; kb < W; kb += U) {
        if (w0 + kb >= nmax) break;
        int c[U], vi[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = kb + u;  // compile-time: register selects are static
          c[u] = __shfl_sync(0xffffffffu, mc[idx / TPR], gbase + idx % TPR);
          if constexpr (kSym) vi[u] = __shfl_sync(0xffffffffu, mv[idx / TPR], gbase + idx % TPR);
          else vi[u] = rs + w0 + idx;
        }
        VecD<V> av[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (kPadZero) {
#pragma unroll
            for (int j = 0; j < V; ++j) av[u].v[j] = xv[u].v[j] = 0.0;
          }
          if (w0 + kb + u < n) {
            av[u] = ld_stream_hint<V>(values + (size_t)vi[u] * S + lane0, pol);
            xv[u] = ld_vec<V>(x + (size_t)c[u] * S + lane0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (kPadZero || w0 + kb + u < n) {
#pragma unroll
            for (int j = 0; j < V; ++j) sum.v[j] = EP_DADD(sum.v[j], EP_DMUL(av[u].v[j], xv[u].v[j]));
          }
        }
      }
    }
    return sum;
  }
}

// Variants (ENPROP_OPT_SPMV_VARIANT), batch U entries / min CTAs per SM:
// 0: 4/4; 1: 4/4 + next pass's index window loaded before this pass; 2: 8/2;
// 3: 8/2 + index prefetch; 4: 4/4 with entries past the row end entering the
// sum as +0.0 * +0.0 instead of predicated off (bitwise identical: the running
// sum starts at +0.0, so it is never -0.0 and sum + 0.0 == sum); 5: 8/3;
// 6: 16/1.
template <int kVar>
struct SpmvVariant {
  static constexpr bool kPrefetch = kVar == 1 || kVar == 3;
  static constexpr bool kPadZero = kVar == 4;
  static constexpr int U = (kVar == 2 || kVar == 3 || kVar == 5) ? 8 : (kVar == 6 ? 16 : 4);
  static constexpr int kMinBlocks = kVar == 5 ? 3 : (kVar == 6 ? 1 : ((kVar & 2) ? 2 : 4));
};

template <int S, bool kTiles, bool kSym, int kVar>
__global__ void __launch_bounds__(256, SpmvVariant<kVar>::kMinBlocks) k_cg_spmv_warp(
    const TileMap tm, const int* __restrict__ row_map, const int* __restrict__ col_entry,
    const double* __restrict__ values, const double* __restrict__ p_new, double* __restrict__ q,
    const double* __restrict__ p_gather, const int* __restrict__ vpos, const FinArgs f) {
  EP_PDL_ENTRY();
  using Sh = WarpTile<S>;
  using Var = SpmvVariant<kVar>;
  constexpr int V = Sh::V, TPR = Sh::TPR, R = Sh::R;
  if (f.cg->done) return;
  const uint64_t pol = l2_policy_evict_normal();
  const int lane = threadIdx.x & 31;
  const int g = lane / TPR, sub = lane % TPR;
  const int lane0 = sub * V;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // tile (or 16-row chunk) of this thread and its first row / row count
  const int unit = warp * Sh::TILES + (Sh::TILES > 1 ? g / kTileRows : 0);
  int r0, nr;
  if constexpr (kTiles) {
    if (unit < tm.num_tiles()) tm.tile(unit, r0, nr);
    else r0 = 0, nr = 0;
  } else {
    r0 = unit * kTileRows;
    nr = imin(kTileRows, tm.rows - r0);
  }
  const int g16 = Sh::TILES > 1 ? g % kTileRows : g;  // row within the tile at pass 0
  // HALF > 0: the top tree level (h = 8 >= R) pairs pass ps with ps + HALF and
  // is applied as soon as pass ps + HALF is known (fewer live registers).
  constexpr int HALF = Sh::PASSES / 2;
  double prod[HALF > 0 ? HALF : 1][V];
  RowIdx<S> ix;
  if constexpr (Var::kPrefetch)
    row_index<S, kSym>(g16 < nr ? r0 + g16 : -1, row_map, col_entry, vpos, sub, pol, ix);
#pragma unroll
  for (int ps = 0; ps < Sh::PASSES; ++ps) {
    const int tr = ps * R + g16;
    const int row = tr < nr ? r0 + tr : -1;
    RowIdx<S> rix;
    if constexpr (Var::kPrefetch) {
      rix = ix;
      if (ps + 1 < Sh::PASSES) {
        const int tn = tr + R;
        row_index<S, kSym>(tn < nr ? r0 + tn : -1, row_map, col_entry, vpos, sub, pol, ix);
      }
    } else {
      row_index<S, kSym>(row, row_map, col_entry, vpos, sub, pol, rix);
    }
    const VecD<V> sum = row_compute<S, kSym, Var::U, Var::kPadZero>(row, rix, row_map, col_entry, values, p_gather,
                                                     vpos, sub, pol);
    double cur[V];
#pragma unroll
    for (int j = 0; j < V; ++j) cur[j] = 0.0;
    if (row >= 0) {
      st_vec<V>(q + (size_t)row * S + lane0, sum);
      if constexpr (kTiles) {
        const VecD<V> pn = ld_vec<V>(p_new + (size_t)row * S + lane0);
#pragma unroll
        for (int j = 0; j < V; ++j) cur[j] = EP_DMUL(pn.v[j], sum.v[j]);
      } else if (f.prod) {  // serial order: p*q for the chain kernel (kernels.hpp:67)
        const VecD<V> pn = ld_vec<V>(p_new + (size_t)row * S + lane0);
        VecD<V> pq;
#pragma unroll
        for (int j = 0; j < V; ++j) pq.v[j] = EP_DMUL(pn.v[j], sum.v[j]);
        st_vec<V>(f.prod + (size_t)row * S + lane0, pq);
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (HALF == 0) prod[0][j] = cur[j];
      else if (ps < HALF) prod[ps % (HALF > 0 ? HALF : 1)][j] = cur[j];
      else prod[(ps - HALF) % (HALF > 0 ? HALF : 1)][j] = EP_DADD(prod[(ps - HALF) % (HALF > 0 ? HALF : 1)][j], cur[j]);
    }
  }
  if constexpr (kTiles) {
    // remaining register levels h with R <= h < 8: rows r and r+h are slots ps, ps + h/R
#pragma unroll
    for (int h = kTileRows / 4; h >= R && h >= 1; h >>= 1)
#pragma unroll
      for (int ps = 0; ps < h / R; ++ps)
#pragma unroll
        for (int j = 0; j < V; ++j) prod[ps][j] = EP_DADD(prod[ps][j], prod[ps + h / R][j]);
    // levels h < R: row g16 + h lives h*TPR lanes up
#pragma unroll
    for (int h = (R < kTileRows ? R : kTileRows) / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const double o = __shfl_down_sync(0xffffffffu, prod[0][j], h * TPR);
        prod[0][j] = EP_DADD(prod[0][j], o);
      }
    if (g16 == 0 && nr > 0) {
#pragma unroll
      for (int j = 0; j < V; ++j) f.partials[(size_t)unit * S + lane0 + j] = prod[0][j];
    }
  }
}

// Direction pass (split variant), every row:
//   x     = alpha_prev*p_old + x   on lanes that owe it (pcg.hpp:94, deferred
//                                  from the previous iteration's update)
//   p_new = 1.0*r + beta*p_old     (pcg.hpp:101; p_new = r when it == 0)
// Both are the reference's operations on the same operands, only scheduled
// where p_old is read anyway, which saves one vector pass per iteration.
constexpr int kDirPasses = 2;

template <int S, int NT>
__global__ void __launch_bounds__(NT, 65536 / (NT * 48)) k_cg_direction(int rows, const double* __restrict__ r,
                                                      const double* __restrict__ p_old,
                                                      double* __restrict__ p_new,
                                                      double* __restrict__ x,
                                                      const CgState* __restrict__ cg) {
  EP_PDL_ENTRY();
  constexpr int P = kDirPasses;
  using Sh = TileShape<S, P, NT>;
  constexpr int V = Sh::V;
  if (cg->done) return;
  const bool first = cg->it == 0;
  const int lane0 = (threadIdx.x % Sh::TPR) * V;
  VecD<V> beta;
  double al[V];
  bool pend[V];
  bool any = false;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    beta.v[j] = cg->beta[lane0 + j];
    al[j] = cg->alpha[lane0 + j];
    pend[j] = !first && cg->pending[lane0 + j] != 0;
    any |= pend[j];
  }
  VecD<V> rv[P], pv[P], xv[P];
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    const int row = blockIdx.x * Sh::ROWS + ps * Sh::RPC + threadIdx.x / Sh::TPR;
    if (row < rows) {
      rv[ps] = ld_vec<V>(r + (size_t)row * S + lane0);
      if (!first) pv[ps] = ld_vec<V>(p_old + (size_t)row * S + lane0);
      if (any) xv[ps] = ld_vec<V>(x + (size_t)row * S + lane0);
    }
  }
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    const int row = blockIdx.x * Sh::ROWS + ps * Sh::RPC + threadIdx.x / Sh::TPR;
    if (row < rows) {
      VecD<V> pn = rv[ps];
      if (!first) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          pn.v[j] = EP_DADD(pn.v[j], EP_DMUL(beta.v[j], pv[ps].v[j]));
          if (pend[j]) xv[ps].v[j] = EP_DADD(EP_DMUL(al[j], pv[ps].v[j]), xv[ps].v[j]);
        }
      }
      st_vec<V>(p_new + (size_t)row * S + lane0, pn);
      if (any) st_vec<V>(x + (size_t)row * S + lane0, xv[ps]);
    }
  }
}

// After the loop: x = alpha*p_last + x on lanes still owing it (p_last is the
// p of iteration it-1, i.e. buffer p[it & 1]).
template <int S>
__global__ void __launch_bounds__(256) k_cg_flush(int rows, double* __restrict__ x,
                                                  const double* __restrict__ p0,
                                                  const double* __restrict__ p1,
                                                  const CgState* __restrict__ cg) {
  EP_PDL_ENTRY();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)rows * S) return;
  const int e = (int)(g % S);
  if (!cg->pending[e]) return;
  const double* p = (cg->it & 1) ? p1 : p0;
  x[g] = EP_DADD(EP_DMUL(cg->alpha[e], p[g]), x[g]);
}

template <int S>
static cudaError_t cg_flush_s(int rows, double* x, double* const* p, const CgState* cg,
                              cudaStream_t st) {
  const int64_t t = (int64_t)rows * S;
  if (t == 0) return cudaSuccess;
  launch_kk(16, k_cg_flush<S>, dim3((int)((t + 255) / 256)), dim3(256), 0, st, rows, x, p[0], p[1], cg);
  return cudaGetLastError();
}

cudaError_t launch_cg_flush(int s, int rows, double* x, double* const* p, const CgState* cg,
                            cudaStream_t st) {
  EP_DISPATCH_S(s, cg_flush_s, rows, x, p, cg, st);
}

template <int S>
static cudaError_t cg_direction_s(int rows, const double* r, const double* p_old, double* p_new,
                                  double* x, const CgState* cg, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (vec_nt() == 128) {
    using Sd = TileShape<S, kDirPasses, 128>;
    launch_kk(1, k_cg_direction<S, 128>, dim3((rows + Sd::ROWS - 1) / Sd::ROWS), dim3(128), 0, st, rows, r, p_old, p_new, x, cg);
  } else {
    using Sd = TileShape<S, kDirPasses, 256>;
    launch_kk(1, k_cg_direction<S, 256>, dim3((rows + Sd::ROWS - 1) / Sd::ROWS), dim3(256), 0, st, rows, r, p_old, p_new, x, cg);
  }
  return cudaGetLastError();
}

cudaError_t launch_cg_direction(int s, int rows, const double* r, const double* p_old,
                                double* p_new, double* x, const CgState* cg, cudaStream_t st) {
  EP_DISPATCH_S(s, cg_direction_s, rows, r, p_old, p_new, x, cg, st);
}

template <int S>
static cudaError_t cg_spmv_s(bool tiles, bool fused_dir, bool run_direction, const TileMap& tm,
                             const int* row_map,
                             const int* col_entry, const double* values, const double* r,
                             const double* p_old, double* p_new, double* q, double* x,
                             const double* p_gather, const int* vpos, const FinArgs& f,
                             cudaStream_t st) {
  using Sh = TileShape<S, 1>;
  const int blocks = tiles ? (tm.num_tiles() + Sh::TPC - 1) / Sh::TPC : (tm.rows + Sh::ROWS - 1) / Sh::ROWS;
  if (blocks == 0) return cudaSuccess;
  if (!fused_dir && run_direction) {  // else the caller ran the direction pass (+ halo)
    using Sd = TileShape<S, kDirPasses, 256>;
    launch_kk(1, k_cg_direction<S, 256>, dim3((tm.rows + Sd::ROWS - 1) / Sd::ROWS), dim3(256), 0, st, tm.rows, r, p_old, p_new, x, f.cg);
  }
#define EP_CG_SPMV(T, D, Y)                                                                   \
  launch_kk(2, k_cg_spmv<S, T, D, Y>, dim3(blocks), dim3(256), 0, st, tm, row_map, col_entry, values, r, p_old, p_new, q, \
                                                x, p_gather, vpos, f)
  if (!fused_dir) {  // warp-per-tile kernel (split direction schedule)
    using Sw = WarpTile<S>;
    const int units = tiles ? tm.num_tiles() : (tm.rows + kTileRows - 1) / kTileRows;
    const int warps = (units + Sw::TILES - 1) / Sw::TILES;
    const int wblocks = (warps + 7) / 8;
#define EP_CG_SPMV_W(T, Y, K)                                                                 \
  launch_kk(2, k_cg_spmv_warp<S, T, Y, K>, dim3(wblocks), dim3(256), 0, st, tm, row_map, col_entry, values, p_new, q, \
                                                      p_gather, vpos, f)
    // auto: 8-entry batches at 2 CTAs/SM for symmetric storage, 4 at 4 CTAs/SM
    // for full storage (same-process A/B at 64^3, s = 32: 0.301 vs 0.332 ms and
    // 0.366 vs 0.391 ms; tools/kernel_bench.py --ab)
    const int var = spmv_variant() >= 0 ? spmv_variant() : (vpos ? 2 : 0);
#define EP_CG_SPMV_WV(T, Y)                 \
  switch (var) {                            \
    case 1: EP_CG_SPMV_W(T, Y, 1); break;   \
    case 2: EP_CG_SPMV_W(T, Y, 2); break;   \
    case 3: EP_CG_SPMV_W(T, Y, 3); break;   \
    case 4: EP_CG_SPMV_W(T, Y, 4); break;   \
    case 5: EP_CG_SPMV_W(T, Y, 5); break;   \
    case 6: EP_CG_SPMV_W(T, Y, 6); break;   \
    default: EP_CG_SPMV_W(T, Y, 0); break;  \
  }
    if (vpos) {
      if (tiles) EP_CG_SPMV_WV(true, true)
      else EP_CG_SPMV_WV(false, true)
    } else {
      if (tiles) EP_CG_SPMV_WV(true, false)
      else EP_CG_SPMV_WV(false, false)
    }
#undef EP_CG_SPMV_WV
#undef EP_CG_SPMV_W
    return cudaGetLastError();
  }
  if (vpos) {  // symmetric storage: split direction schedule only
    if (fused_dir) return cudaErrorInvalidValue;
    if (tiles) EP_CG_SPMV(true, false, true);
    else EP_CG_SPMV(false, false, true);
  } else if (tiles) {
    if (fused_dir) EP_CG_SPMV(true, true, false);
    else EP_CG_SPMV(true, false, false);
  } else {
    if (fused_dir) EP_CG_SPMV(false, true, false);
    else EP_CG_SPMV(false, false, false);
  }
#undef EP_CG_SPMV
  return cudaGetLastError();
}

cudaError_t launch_cg_spmv(int s, bool tiles, bool fused_dir, bool run_direction,
                           const TileMap& tm, const int* row_map, const int* col_entry,
                           const double* values, const double* r, const double* p_old,
                           double* p_new, double* q, double* x, const double* p_gather,
                           const int* vpos, const FinArgs& f, cudaStream_t st) {
  EP_DISPATCH_S(s, cg_spmv_s, tiles, fused_dir, run_direction, tm, row_map, col_entry, values, r,
                p_old, p_new, q, x, p_gather, vpos, f, st);
}

// r = (-alpha)*q + 1.0*r on active lanes (pcg.hpp:95 via axpby,
// kernels.hpp:84: 1.0*y is exact); r.r for the next dot.  P rows per thread,
// all loads issued before any arithmetic.  (x is updated one pass later, in
// k_cg_direction / k_cg_flush.)
template <int S, bool kTiles, int NT>
__global__ void __launch_bounds__(NT, 65536 / (NT * 48)) k_cg_update(const TileMap tm, double* __restrict__ r,
                                                   const double* __restrict__ q, const FinArgs f) {
  EP_PDL_ENTRY();
  constexpr int P = NT == 128 ? 2 : kStreamPasses;  // 48-register cap at 128 threads
  using Sh = TileShape<S, P, NT>;
  constexpr int V = Sh::V;
  const CgState* cg = f.cg;
  if (cg->done) return;
  __shared__ double sprod[kTiles ? Sh::ROWS * S : 1];
  const int lane0 = (threadIdx.x % Sh::TPR) * V;
  double al[V];
  bool act[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    al[j] = cg->alpha[lane0 + j];
    act[j] = cg->active[lane0 + j] != 0;
  }
  int row[P];
  VecD<V> rv[P], qv[P];
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    row[ps] = cg_row<S, P, kTiles, NT>(tm, ps * Sh::RPC + threadIdx.x / Sh::TPR);
    if (row[ps] >= 0) {
      const size_t off = (size_t)row[ps] * S + lane0;
      rv[ps] = ld_vec<V>(r + off);
      qv[ps] = ld_vec<V>(q + off);
    }
  }
#pragma unroll
  for (int ps = 0; ps < P; ++ps) {
    const int slot = ps * Sh::RPC + threadIdx.x / Sh::TPR;
    VecD<V> pr;
    if (row[ps] >= 0) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (act[j]) rv[ps].v[j] = EP_DADD(EP_DMUL(-al[j], qv[ps].v[j]), rv[ps].v[j]);
        pr.v[j] = EP_DMUL(rv[ps].v[j], rv[ps].v[j]);
      }
      st_vec<V>(r + (size_t)row[ps] * S + lane0, rv[ps]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) pr.v[j] = 0.0;
    }
    if constexpr (kTiles) {
#pragma unroll
      for (int j = 0; j < V; ++j) sprod[slot * S + lane0 + j] = pr.v[j];
    }
  }
  if constexpr (kTiles) tiles_finish<S, P, NT>(tm, sprod, f);
}

template <int S, int NT>
static cudaError_t cg_update_nt(bool tiles, const TileMap& tm, double* r, const double* q,
                                const FinArgs& f, cudaStream_t st) {
  using Sh = TileShape<S, NT == 128 ? 2 : kStreamPasses, NT>;
  const int blocks = tiles ? (tm.num_tiles() + Sh::TPC - 1) / Sh::TPC : (tm.rows + Sh::ROWS - 1) / Sh::ROWS;
  if (blocks == 0) return cudaSuccess;
  if (tiles) launch_kk(8, k_cg_update<S, true, NT>, dim3(blocks), dim3(NT), 0, st, tm, r, q, f);
  else launch_kk(8, k_cg_update<S, false, NT>, dim3(blocks), dim3(NT), 0, st, tm, r, q, f);
  return cudaGetLastError();
}

template <int S>
static cudaError_t cg_update_s(bool tiles, const TileMap& tm, double* r, const double* q,
                               const FinArgs& f, cudaStream_t st) {
  if (vec_nt() == 128) return cg_update_nt<S, 128>(tiles, tm, r, q, f, st);
  return cg_update_nt<S, 256>(tiles, tm, r, q, f, st);
}

cudaError_t launch_cg_update(int s, bool tiles, const TileMap& tm, double* r, const double* q,
                             const FinArgs& f, cudaStream_t st) {
  EP_DISPATCH_S(s, cg_update_s, tiles, tm, r, q, f, st);
}

// =============================================================================
// Symmetric storage. The assembled matrix is exactly symmetric
// (G_qij == G_qji bitwise; Dirichlet keeps symmetry), so the device-resident
// pipeline stores row r's entries with col >= r only ("upper", diagonal
// included, in column order): nnz_up = (nnz + rows)/2 for a structurally
// symmetric graph. vpos[k] maps every entry of the full CRS to its slot.
// =============================================================================
// Graph row r has coordinate r - base (a slab's store rows: `base` ghost rows
// before the owned ones; columns are in owned coordinates); base = 0 on one GPU.
__global__ void k_sym_count(int rows, int base, const int* __restrict__ row_map,
                            const int* __restrict__ col_entry, int* __restrict__ cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int c = 0;
  for (int k = row_map[r]; k < row_map[r + 1]; ++k) c += col_entry[k] >= r - base;
  cnt[r] = c;
}

// first k in [lo, hi) with col_entry[k] >= v
__device__ __forceinline__ int lower_bound_i(const int* a, int lo, int hi, int v) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_sym_vpos(int rows, int base, const int* __restrict__ row_map,
                           const int* __restrict__ col_entry, const int* __restrict__ up_start,
                           int* __restrict__ vpos, int* __restrict__ bad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int rc = r - base;  // this row's coordinate
  const int rs = row_map[r], re = row_map[r + 1];
  const int first_up = lower_bound_i(col_entry, rs, re, rc);
  for (int k = rs; k < re; ++k) {
    const int c = col_entry[k];
    if (c >= rc) {
      vpos[k] = up_start[r] + (k - first_up);
    } else {  // transposed entry (c, r) in row c's upper part
      const int cr = c + base;  // graph row of column c
      if (cr < 0) {             // a ghost row's lower entry: never read
        if (r >= base) atomicAdd(bad, 1);
        vpos[k] = -1;
        continue;
      }
      const int cs = row_map[cr], ce = row_map[cr + 1];
      const int fu = lower_bound_i(col_entry, cs, ce, c);
      const int t = lower_bound_i(col_entry, fu, ce, rc);
      if (t >= ce || col_entry[t] != rc) {
        atomicAdd(bad, 1);  // pattern not symmetric
        vpos[k] = 0;
      } else {
        vpos[k] = up_start[cr] + (t - fu);
      }
    }
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_sym_expand(int64_t nnz, const int* __restrict__ vpos,
                                                    const double* __restrict__ up,
                                                    double* __restrict__ full) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nnz * S) return;
  const int64_t k = g / S;
  full[g] = up[(int64_t)vpos[k] * S + (g - k * S)];
}

template <int S>
static cudaError_t sym_expand_s(int64_t nnz, const int* vpos, const double* up, double* full,
                                cudaStream_t st) {
  const int64_t t = nnz * S;
  if (t == 0) return cudaSuccess;
  k_sym_expand<S><<<(int)((t + 255) / 256), 256, 0, st>>>(nnz, vpos, up, full);
  return cudaGetLastError();
}

cudaError_t launch_sym_expand(int s, int64_t nnz, const int* vpos, const double* up, double* full,
                              cudaStream_t st) {
  EP_DISPATCH_S(s, sym_expand_s, nnz, vpos, up, full, st);
}

}  // namespace ep

#include <cub/device/device_scan.cuh>

namespace ep {

cudaError_t build_sym(int rows, const int* row_map, const int* col_entry, int* vpos,
                      int64_t* nnz_up, cudaStream_t st, int* up_start, int base) {
  int *cnt = nullptr, *start = nullptr, *bad = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t err = cudaMalloc(&cnt, (size_t)(rows + 1) * sizeof(int));
  if (err == cudaSuccess) err = cudaMalloc(&start, (size_t)(rows + 1) * sizeof(int));
  if (err == cudaSuccess) err = cudaMalloc(&bad, sizeof(int));
  if (err == cudaSuccess) err = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (err == cudaSuccess) err = cudaMemsetAsync(cnt + rows, 0, sizeof(int), st);
  if (err == cudaSuccess && rows > 0) {
    k_sym_count<<<(rows + 255) / 256, 256, 0, st>>>(rows, base, row_map, col_entry, cnt);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess) err = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, start, rows + 1, st);
  if (err == cudaSuccess) err = cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 8);
  if (err == cudaSuccess) err = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, start, rows + 1, st);
  if (err == cudaSuccess && rows > 0) {
    k_sym_vpos<<<(rows + 255) / 256, 256, 0, st>>>(rows, base, row_map, col_entry, start, vpos, bad);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess && up_start)
    err = cudaMemcpyAsync(up_start, start, (size_t)(rows + 1) * sizeof(int), cudaMemcpyDeviceToDevice, st);
  int h_total = 0, h_bad = 0;
  if (err == cudaSuccess) err = cudaMemcpyAsync(&h_total, start + rows, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  cudaFree(cnt);
  cudaFree(start);
  cudaFree(bad);
  cudaFree(tmp);
  if (err == cudaSuccess && h_bad) err = cudaErrorInvalidValue;
  *nnz_up = h_total;
  return err;
}

}  // namespace ep
