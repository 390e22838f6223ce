// enprop_b200 assembly kernels for sm_100a: ensemble Q1 FEM assembly with a
// KL diffusion field (proj/include/enprop/fem.hpp:115-202) and the symmetric
// Dirichlet elimination (fem.hpp:218-243), bitwise equal to the reference.
#include "ep_common.cuh"
#include "ep_kernels.h"

namespace ep {

// =============================================================================
// Assembly: node-centric gather (fem.hpp:115-202 + apply_dirichlet :218-243).
//
// The reference scatters element matrices cell by cell in ascending cell id,
// so global entry (P,Q) = 0.0 + A_c1[P][Q] + A_c2[P][Q] + ... over the cells
// containing both nodes in ascending id.  Here one thread owns one
// (row P, sample e): it walks the <= 8 cells around P in ascending id
// (dk, dj, di in {-1,0}, ck-major), rebuilds row P's part of each element
// matrix with the reference's operation order, and adds it into 27 register
// accumulators (one per stencil slot).  Each value is produced by exactly one
// thread and written once: no atomics, bitwise equal to the reference.
//
// kNonlinear = false is the alpha = beta = 0 path: the advection and reaction
// terms are exact signed zeros there and adding them changes no bit
// (DESIGN.md §3).  kHasU = false is u = 0: every element residual is then an
// exact +0.0 (sums of signed zeros starting from +0.0), so the residual before
// Dirichlet is +0.0 and only the Jacobian is formed.
// =============================================================================
template <int S, bool kNonlinear, bool kHasU>
__global__ void __launch_bounds__(256) k_assemble(const __grid_constant__ AsmArgs a) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int lrow = gt / S;  // local row
  const int row = a.row_begin + lrow;  // global node id
  const int e = gt - lrow * S;
  if (lrow >= a.rows) return;
  const int n = a.n, N = n + 1, n2 = 2 * n;
  const int i = row % N, j = (row / N) % N, k = row / (N * N);
  const AsmTables& T = a.T;  // kernel parameter: uniform constant-bank reads
  const double wd = T.wd;

  double acc[27];
#pragma unroll
  for (int t = 0; t < 27; ++t) acc[t] = 0.0;
  double res = 0.0;

#pragma unroll
  for (int dk = -1; dk <= 0; ++dk)
#pragma unroll
    for (int dj = -1; dj <= 0; ++dj)
#pragma unroll
      for (int di = -1; di <= 0; ++di) {
        const int ci = i + di, cj = j + dj, ck = k + dk;
        if (ci < 0 || ci >= n || cj < 0 || cj >= n || ck < a.kc_lo || ck >= n) continue;
        const int iloc = (-di) | ((-dj) << 1) | ((-dk) << 2);  // row P's corner in the cell

        // kappa at the 8 Gauss points (kl.hpp:67-81): kappa = mean, then for each
        // mode t: kappa += (((sigma*sqrt(lambda_t)) * f_ax) * f_ay) * f_az * y_t.
        // The products are shared across points with the same axis bits.
        double kap[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) kap[q] = a.mean;
        for (int t = 0; t < a.m; ++t) {
          const double* Fx = a.F + a.mode_axes[t][0] * n2 + 2 * ci;
          const double* Fy = a.F + a.mode_axes[t][1] * n2 + 2 * cj;
          const double* Fz = a.F + a.mode_axes[t][2] * n2 + 2 * ck;
          const double sl = a.mode_sl[t];
          const double yt = a.y[t * S + e];
          const double fx0 = EP_DMUL(sl, __ldg(Fx)), fx1 = EP_DMUL(sl, __ldg(Fx + 1));
          const double fy0 = __ldg(Fy), fy1 = __ldg(Fy + 1);
          const double fz0 = __ldg(Fz), fz1 = __ldg(Fz + 1);
          const double f00 = EP_DMUL(fx0, fy0), f10 = EP_DMUL(fx1, fy0);
          const double f01 = EP_DMUL(fx0, fy1), f11 = EP_DMUL(fx1, fy1);
          const double fq[8] = {EP_DMUL(f00, fz0), EP_DMUL(f10, fz0), EP_DMUL(f01, fz0),
                                EP_DMUL(f11, fz0), EP_DMUL(f00, fz1), EP_DMUL(f10, fz1),
                                EP_DMUL(f01, fz1), EP_DMUL(f11, fz1)};
#pragma unroll
          for (int q = 0; q < 8; ++q) kap[q] = EP_DADD(kap[q], EP_DMUL(fq[q], yt));
        }

        double ue[8];
        if constexpr (kHasU) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int node =
                (ci + (c & 1)) + N * ((cj + ((c >> 1) & 1)) + N * (ck + ((c >> 2) & 1)));
            ue[c] = a.u[(size_t)(node - a.u_shift) * S + e];
          }
        }

        double ej[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) ej[jj] = 0.0;
        double er = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double kappa = kap[q];
          double rdv = 0.0;
          if constexpr (kHasU) {
            double uq = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;  // fem.hpp:160-166
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              uq = EP_DADD(uq, EP_DMUL(T.VAL[q][c], ue[c]));
              gx = EP_DADD(gx, EP_DMUL(T.GS[q][c][0], ue[c]));
              gy = EP_DADD(gy, EP_DMUL(T.GS[q][c][1], ue[c]));
              gz = EP_DADD(gz, EP_DMUL(T.GS[q][c][2], ue[c]));
            }
            const double adv =  // fem.hpp:167
                EP_DMUL(T.alpha, EP_DADD(EP_DADD(EP_DMUL(T.vx, gx), EP_DMUL(T.vy, gy)),
                                         EP_DMUL(T.vz, gz)));
            const double rea = EP_DMUL(T.beta, EP_DMUL(uq, uq));  // fem.hpp:168
            rdv = EP_DMUL(EP_DMUL(2.0, T.beta), uq);              // fem.hpp:169
            const double ni = T.VAL[q][iloc];                     // fem.hpp:177-180
            double t1 = EP_DMUL(kappa, EP_DADD(EP_DADD(EP_DMUL(gx, T.GS[q][iloc][0]),
                                                       EP_DMUL(gy, T.GS[q][iloc][1])),
                                               EP_DMUL(gz, T.GS[q][iloc][2])));
            t1 = EP_DADD(t1, EP_DMUL(adv, ni));
            t1 = EP_DADD(t1, EP_DMUL(rea, ni));
            er = EP_DADD(er, EP_DMUL(wd, t1));
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {  // fem.hpp:189-191
            double t2 = EP_DMUL(kappa, T.G[q][iloc][jj]);
            if constexpr (kNonlinear) {
              t2 = EP_DADD(t2, T.ADV[q][iloc][jj]);
              t2 = EP_DADD(t2, EP_DMUL(rdv, T.NN[q][iloc][jj]));
            }
            ej[jj] = EP_DADD(ej[jj], EP_DMUL(wd, t2));
          }
        }
        if constexpr (kHasU) res = EP_DADD(res, er);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int ox = di + (jj & 1), oy = dj + ((jj >> 1) & 1), oz = dk + ((jj >> 2) & 1);
          const int slot = (oz + 1) * 9 + (oy + 1) * 3 + (ox + 1);
          acc[slot] = EP_DADD(acc[slot], ej[jj]);
        }
      }

  // apply_dirichlet (fem.hpp:218-243), row-local so it fuses exactly.
  if (a.dirichlet) {
    if (i == 0 || i == n) {
#pragma unroll
      for (int t = 0; t < 27; ++t) acc[t] = (t == 13) ? 1.0 : 0.0;
      const double ur = kHasU ? a.u[(size_t)(row - a.u_shift) * S + e] : 0.0;
      res = EP_DSUB(ur, i == 0 ? a.bc0 : a.bc1);
    } else {
#pragma unroll
      for (int t = 0; t < 27; ++t) {
        const int ox = t % 3 - 1, oy = (t / 3) % 3 - 1, oz = t / 9 - 1;
        const int ii = i + ox, jj = j + oy, kk = k + oz;
        if (jj < 0 || jj >= N || kk < a.kc_lo || kk >= N) continue;
        if (ii == 0 || ii == n) {
          const double g = ii == 0 ? a.bc0 : a.bc1;
          const double uc = kHasU ? a.u[(size_t)(ii + N * (jj + N * kk) - a.u_shift) * S + e] : 0.0;
          res = EP_DADD(res, EP_DMUL(acc[t], EP_DSUB(g, uc)));
          acc[t] = 0.0;
        }
      }
    }
  }

  const int rs = a.row_map[lrow];
  int pos = 0;
#pragma unroll
  for (int t = 0; t < 27; ++t) {
    const int ox = t % 3 - 1, oy = (t / 3) % 3 - 1, oz = t / 9 - 1;
    const int ii = i + ox, jj = j + oy, kk = k + oz;
    if (ii < 0 || ii >= N || jj < 0 || jj >= N || kk < 0 || kk >= N) continue;
    if (a.vpos == nullptr) {
      a.values[(size_t)(rs + pos) * S + e] = acc[t];
    } else if (t >= 13) {  // stencil slots are in column order; slot 13 is the diagonal
      a.values[(size_t)a.vpos[rs + pos] * S + e] = acc[t];
    }
    ++pos;
  }
  a.residual[(size_t)lrow * S + e] = res;
}

template <int S>
static cudaError_t assemble_s(const AsmArgs& a, cudaStream_t st) {
  const int64_t threads = (int64_t)a.rows * S;
  const int grid = (int)((threads + 255) / 256);
  const bool has_u = a.u != nullptr;
  if (a.nonlinear) {
    if (has_u) k_assemble<S, true, true><<<grid, 256, 0, st>>>(a);
    else k_assemble<S, true, false><<<grid, 256, 0, st>>>(a);
  } else {
    if (has_u) k_assemble<S, false, true><<<grid, 256, 0, st>>>(a);
    else k_assemble<S, false, false><<<grid, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_assemble(int s, const AsmArgs& a, cudaStream_t st) {
  EP_DISPATCH_S(s, assemble_s, a, st);
}

// =============================================================================
// Standalone apply_dirichlet (fem.hpp:218-243): one thread per (row, sample).
// =============================================================================
template <int S>
__global__ void __launch_bounds__(256) k_dirichlet(int n, double bc0, double bc1,
                                                   const int* __restrict__ row_map,
                                                   const int* __restrict__ col_entry,
                                                   const double* __restrict__ u,
                                                   double* __restrict__ values,
                                                   double* __restrict__ residual) {
  const int N = n + 1;
  const int rows = N * N * N;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt / S, e = gt - row * S;
  if (row >= rows) return;
  const int rx = row % N;
  const int rs = row_map[row], re = row_map[row + 1];
  if (rx == 0 || rx == n) {
    for (int k = rs; k < re; ++k) values[(size_t)k * S + e] = (col_entry[k] == row) ? 1.0 : 0.0;
    const double ur = u ? u[(size_t)row * S + e] : 0.0;
    residual[(size_t)row * S + e] = EP_DSUB(ur, rx == 0 ? bc0 : bc1);
  } else {
    double res = residual[(size_t)row * S + e];
    for (int k = rs; k < re; ++k) {
      const int col = col_entry[k];
      const int cx = col % N;
      if (cx == 0 || cx == n) {
        const double g = cx == 0 ? bc0 : bc1;
        const double uc = u ? u[(size_t)col * S + e] : 0.0;
        res = EP_DADD(res, EP_DMUL(values[(size_t)k * S + e], EP_DSUB(g, uc)));
        values[(size_t)k * S + e] = 0.0;
      }
    }
    residual[(size_t)row * S + e] = res;
  }
}

template <int S>
static cudaError_t dirichlet_s(int n, double bc0, double bc1, const int* row_map,
                               const int* col_entry, const double* u, double* values,
                               double* residual, cudaStream_t st) {
  const int64_t rows = (int64_t)(n + 1) * (n + 1) * (n + 1);
  const int grid = (int)((rows * S + 255) / 256);
  k_dirichlet<S><<<grid, 256, 0, st>>>(n, bc0, bc1, row_map, col_entry, u, values, residual);
  return cudaGetLastError();
}

cudaError_t launch_dirichlet(int s, int n, double bc0, double bc1, const int* row_map,
                             const int* col_entry, const double* u, double* values,
                             double* residual, cudaStream_t st) {
  EP_DISPATCH_S(s, dirichlet_s, n, bc0, bc1, row_map, col_entry, u, values, residual, st);
}

}  // namespace ep
