/* TEST INFRASTRUCTURE ONLY — see enprop_oracle.h.
 * Each function restates the cited reference code (paths relative to
 * /root/reference/) without copying it: plain C, explicit loops, the same
 * left-to-right floating-point order. Built with -ffp-contract=off. */
#include "enprop_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the C++ std engine used by proj/src/samples.cpp:8) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* proj/src/samples.cpp:7-18: top 53 bits -> [0,1) -> [-1,1) */
void or_draw_samples(uint64_t seed, int count, int m, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < m; ++j)
      out[(size_t)i * m + j] = (double)(mt64_next(&g) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

/* ------------------------------------------------------------------------ */
/* proj/src/mesh.cpp:13-55: 27-point node adjacency, columns ascending
 * (kk -> jj -> ii), node id = i + N(j + N k) (mesh.hpp:24-26). */
int64_t or_graph_nnz(int n) {
  int64_t t = 3 * (int64_t)(n + 1) - 2;
  return t * t * t;
}

void or_build_graph(int n, int* row_map, int* col_entry) {
  const int N = n + 1;
  int at = 0;
  row_map[0] = 0;
  for (int k = 0; k < N; ++k)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i) {
        const int ilo = i > 0 ? i - 1 : 0, ihi = i < N - 1 ? i + 1 : N - 1;
        const int jlo = j > 0 ? j - 1 : 0, jhi = j < N - 1 ? j + 1 : N - 1;
        const int klo = k > 0 ? k - 1 : 0, khi = k < N - 1 ? k + 1 : N - 1;
        for (int kk = klo; kk <= khi; ++kk)
          for (int jj = jlo; jj <= jhi; ++jj)
            for (int ii = ilo; ii <= ihi; ++ii) col_entry[at++] = ii + N * (jj + N * kk);
        row_map[i + N * (j + N * k) + 1] = at;
      }
}

/* binary search, proj/include/enprop/crs.hpp:114-121 */
static int find_entry(const int* row_map, const int* col_entry, int row, int col) {
  int lo = row_map[row], hi = row_map[row + 1];
  while (lo < hi) {
    int mid = lo + (hi - lo) / 2;
    if (col_entry[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return (lo < row_map[row + 1] && col_entry[lo] == col) ? lo : -1;
}

/* ------------------------------------------------------------------------ */
/* KL field: proj/src/kl.cpp:13-89, proj/include/enprop/kl.hpp:17-81 */
static const double kPi = 3.14159265358979323846;

static double kl_residual(double w, double c, int cosine_branch) {
  /* kl.cpp:13-19 product forms */
  return cosine_branch ? w * sin(0.5 * w) - c * cos(0.5 * w) : c * sin(0.5 * w) + w * cos(0.5 * w);
}

static double kl_bisect(double lo, double hi, double c, int cosine_branch) {
  /* kl.cpp:21-35 */
  double flo = kl_residual(lo, c, cosine_branch);
  while (hi - lo > 1e-12) {
    double mid = 0.5 * (lo + hi);
    double fmid = kl_residual(mid, c, cosine_branch);
    if ((flo < 0.0) == (fmid < 0.0)) {
      lo = mid;
      flo = fmid;
    } else {
      hi = mid;
    }
  }
  return 0.5 * (lo + hi);
}

typedef struct {
  int ax[3];
  double eig, sq;
} kl_cand;

static int kl_cand_cmp(const void* pa, const void* pb) {
  /* kl.cpp:84-87: eigenvalue descending, ties by lexicographic axis triple */
  const kl_cand* p = (const kl_cand*)pa;
  const kl_cand* q = (const kl_cand*)pb;
  if (p->eig != q->eig) return p->eig > q->eig ? -1 : 1;
  for (int a = 0; a < 3; ++a)
    if (p->ax[a] != q->ax[a]) return p->ax[a] < q->ax[a] ? -1 : 1;
  return 0;
}

int or_kl_init(or_kl_field* f, int m, double mean, double sigma, double corr_length) {
  if (m < 1 || m > OR_MAX_TERMS || mean <= 0.0 || sigma < 0.0 || corr_length <= 0.0) return OR_INVALID;
  memset(f, 0, sizeof(*f));
  f->m = m;
  f->mean = mean;
  f->sigma = sigma;
  f->corr_length = corr_length;
  const double c = 1.0 / corr_length;
  for (int t = 0; t < m; ++t) { /* kl.cpp:41-62 */
    const int k = t / 2;
    const int cb = (t % 2 == 0);
    const double lo = cb ? 2 * k * kPi : (2 * k + 1) * kPi;
    const double hi = lo + kPi;
    const double w = kl_bisect(lo, hi, c, cb);
    f->axis_cos[t] = cb;
    f->axis_freq[t] = w;
    f->axis_eig[t] = 2.0 * c / (w * w + c * c);
    const double half_sinc = sin(w) / (2.0 * w);
    f->axis_invnorm[t] = 1.0 / sqrt(cb ? 0.5 + half_sinc : 0.5 - half_sinc);
  }
  const int nc = m * m * m; /* kl.cpp:75-82 */
  kl_cand* cand = (kl_cand*)malloc(sizeof(kl_cand) * (size_t)nc);
  int at = 0;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b)
      for (int d = 0; d < m; ++d) {
        double lambda = f->axis_eig[a] * f->axis_eig[b] * f->axis_eig[d];
        cand[at].ax[0] = a;
        cand[at].ax[1] = b;
        cand[at].ax[2] = d;
        cand[at].eig = lambda;
        cand[at].sq = sqrt(lambda);
        ++at;
      }
  qsort(cand, (size_t)nc, sizeof(kl_cand), kl_cand_cmp);
  for (int i = 0; i < m; ++i) {
    for (int a = 0; a < 3; ++a) f->mode_axes[i][a] = cand[i].ax[a];
    f->mode_eig[i] = cand[i].eig;
    f->mode_sqrt_eig[i] = cand[i].sq;
  }
  free(cand);
  return OR_OK;
}

static double kl_axis_eval(const or_kl_field* f, int t, double x) {
  /* kl.hpp:24-27 */
  const double arg = f->axis_freq[t] * (x - 0.5);
  return (f->axis_cos[t] ? cos(arg) : sin(arg)) * f->axis_invnorm[t];
}

void or_kl_evaluate(const or_kl_field* f, int S, const double x[3], const double* y, double* out) {
  /* kl.hpp:67-81: kappa = mean; kappa += (((sigma*sqrt)*fx)*fy)*fz * y_i */
  for (int e = 0; e < S; ++e) out[e] = f->mean;
  for (int i = 0; i < f->m; ++i) {
    const double factor = f->sigma * f->mode_sqrt_eig[i] * kl_axis_eval(f, f->mode_axes[i][0], x[0]) *
                          kl_axis_eval(f, f->mode_axes[i][1], x[1]) *
                          kl_axis_eval(f, f->mode_axes[i][2], x[2]);
    for (int e = 0; e < S; ++e) out[e] += factor * y[(size_t)i * S + e];
  }
}

/* ------------------------------------------------------------------------ */
/* Q1 basis on 2x2x2 Gauss points: proj/include/enprop/fem.hpp:76-98 */
typedef struct {
  double value[8][8];
  double gradient[8][8][3];
  double offset[8][3];
} basis_tables;

static void make_basis(basis_tables* b) {
  const double g = 1.0 / sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
    for (int a = 0; a < 3; ++a) b->offset[q][a] = 0.5 * (xi[a] + 1.0);
    for (int c = 0; c < 8; ++c) {
      const double sg[3] = {(c & 1) ? 1.0 : -1.0, (c & 2) ? 1.0 : -1.0, (c & 4) ? 1.0 : -1.0};
      const double lin[3] = {0.5 * (1.0 + sg[0] * xi[0]), 0.5 * (1.0 + sg[1] * xi[1]),
                             0.5 * (1.0 + sg[2] * xi[2])};
      b->value[q][c] = lin[0] * lin[1] * lin[2];
      b->gradient[q][c][0] = 0.5 * sg[0] * lin[1] * lin[2];
      b->gradient[q][c][1] = lin[0] * 0.5 * sg[1] * lin[2];
      b->gradient[q][c][2] = lin[0] * lin[1] * 0.5 * sg[2];
    }
  }
}

/* proj/include/enprop/fem.hpp:115-202 — cell loop in ascending cell order,
 * element matrices scatter-added; optional fem.hpp:218-243. */
void or_assemble(int S, int n, const or_kl_field* f, double alpha, double beta,
                 const double velocity[3], const double* u, const double* y, int dirichlet,
                 double bc_x0, double bc_x1, double* values, double* residual) {
  const int N = n + 1;
  const int rows = N * N * N;
  const int64_t nnz = or_graph_nnz(n);
  int* row_map = (int*)malloc(sizeof(int) * (size_t)(rows + 1));
  int* col_entry = (int*)malloc(sizeof(int) * (size_t)nnz);
  or_build_graph(n, row_map, col_entry);
  memset(values, 0, sizeof(double) * (size_t)nnz * S);
  memset(residual, 0, sizeof(double) * (size_t)rows * S);

  basis_tables B;
  make_basis(&B);
  const double h = 1.0 / n;                             /* mesh.hpp:22 */
  const double grad_scale = 2.0 / h;                    /* fem.hpp:135 */
  const double wd = (h / 2.0) * (h / 2.0) * (h / 2.0);  /* fem.hpp:136 */
  const double vx = velocity[0], vy = velocity[1], vz = velocity[2];

  double* ue = (double*)malloc(sizeof(double) * 8 * S);
  double* er = (double*)malloc(sizeof(double) * 8 * S);
  double* ej = (double*)malloc(sizeof(double) * 64 * S);
  double* kappa = (double*)malloc(sizeof(double) * S);
  double* uq = (double*)malloc(sizeof(double) * S * 4);
  double* gxs = uq + S;
  double* gys = uq + 2 * S;
  double* gzs = uq + 3 * S;
  double* tmp = (double*)malloc(sizeof(double) * S * 3);
  double* adv = tmp;
  double* rea = tmp + S;
  double* rdv = tmp + 2 * S;

  for (int cell = 0; cell < n * n * n; ++cell) {
    const int ci = cell % n, cj = (cell / n) % n, ck = cell / (n * n);
    int nodes[8];
    for (int c = 0; c < 8; ++c) /* mesh.hpp:41-49 */
      nodes[c] = (ci + (c & 1)) + N * ((cj + ((c >> 1) & 1)) + N * (ck + ((c >> 2) & 1)));
    for (int c = 0; c < 8; ++c)
      for (int e = 0; e < S; ++e) ue[c * S + e] = u ? u[(size_t)nodes[c] * S + e] : 0.0;
    for (int c = 0; c < 8 * S; ++c) er[c] = 0.0;
    for (int c = 0; c < 64 * S; ++c) ej[c] = 0.0;

    for (int q = 0; q < 8; ++q) {
      const double pt[3] = {(ci + B.offset[q][0]) * h, (cj + B.offset[q][1]) * h,
                            (ck + B.offset[q][2]) * h};
      or_kl_evaluate(f, S, pt, y, kappa);
      for (int e = 0; e < S; ++e) uq[e] = gxs[e] = gys[e] = gzs[e] = 0.0;
      for (int c = 0; c < 8; ++c) {
        const double gsx = B.gradient[q][c][0] * grad_scale;
        const double gsy = B.gradient[q][c][1] * grad_scale;
        const double gsz = B.gradient[q][c][2] * grad_scale;
        for (int e = 0; e < S; ++e) {
          const double uc = ue[c * S + e];
          uq[e] += B.value[q][c] * uc;
          gxs[e] += gsx * uc;
          gys[e] += gsy * uc;
          gzs[e] += gsz * uc;
        }
      }
      for (int e = 0; e < S; ++e) {
        adv[e] = alpha * (vx * gxs[e] + vy * gys[e] + vz * gzs[e]); /* fem.hpp:167 */
        rea[e] = beta * (uq[e] * uq[e]);                           /* fem.hpp:168 */
        rdv[e] = (2.0 * beta) * uq[e];                             /* fem.hpp:169 */
      }
      for (int i = 0; i < 8; ++i) {
        const double gx_i = B.gradient[q][i][0] * grad_scale;
        const double gy_i = B.gradient[q][i][1] * grad_scale;
        const double gz_i = B.gradient[q][i][2] * grad_scale;
        const double n_i = B.value[q][i];
        for (int e = 0; e < S; ++e) /* fem.hpp:177-180 */
          er[i * S + e] += wd * (kappa[e] * (gxs[e] * gx_i + gys[e] * gy_i + gzs[e] * gz_i) +
                                 adv[e] * n_i + rea[e] * n_i);
        for (int j = 0; j < 8; ++j) {
          const double gx_j = B.gradient[q][j][0] * grad_scale;
          const double gy_j = B.gradient[q][j][1] * grad_scale;
          const double gz_j = B.gradient[q][j][2] * grad_scale;
          const double n_j = B.value[q][j];
          const double advect_ij = alpha * (vx * gx_j + vy * gy_j + vz * gz_j) * n_i;
          const double gij = gx_j * gx_i + gy_j * gy_i + gz_j * gz_i;
          const double nn = n_j * n_i;
          for (int e = 0; e < S; ++e) /* fem.hpp:189-191 */
            ej[(i * 8 + j) * S + e] += wd * (kappa[e] * gij + advect_ij + rdv[e] * nn);
        }
      }
    }
    for (int i = 0; i < 8; ++i) { /* fem.hpp:196-200 */
      for (int e = 0; e < S; ++e) residual[(size_t)nodes[i] * S + e] += er[i * S + e];
      for (int j = 0; j < 8; ++j) {
        const int k = find_entry(row_map, col_entry, nodes[i], nodes[j]); /* fem.hpp:52 */
        for (int e = 0; e < S; ++e) values[(size_t)k * S + e] += ej[(i * 8 + j) * S + e];
      }
    }
  }
  if (dirichlet) or_apply_dirichlet(S, n, bc_x0, bc_x1, row_map, col_entry, u, values, residual);
  free(ue); free(er); free(ej); free(kappa); free(uq); free(tmp);
  free(row_map); free(col_entry);
}

/* proj/include/enprop/fem.hpp:218-243 */
void or_apply_dirichlet(int S, int n, double bc_x0, double bc_x1, const int* row_map,
                        const int* col_entry, const double* u, double* values, double* residual) {
  const int N = n + 1;
  const int rows = N * N * N;
  for (int row = 0; row < rows; ++row) {
    const int rx = row % N;
    if (rx == 0 || rx == n) {
      const double g = rx == 0 ? bc_x0 : bc_x1;
      for (int k = row_map[row]; k < row_map[row + 1]; ++k)
        for (int e = 0; e < S; ++e) values[(size_t)k * S + e] = (col_entry[k] == row) ? 1.0 : 0.0;
      for (int e = 0; e < S; ++e)
        residual[(size_t)row * S + e] = (u ? u[(size_t)row * S + e] : 0.0) - g;
    } else {
      for (int k = row_map[row]; k < row_map[row + 1]; ++k) {
        const int col = col_entry[k];
        const int cx = col % N;
        if (cx == 0 || cx == n) {
          const double g = cx == 0 ? bc_x0 : bc_x1;
          for (int e = 0; e < S; ++e) {
            const double uc = u ? u[(size_t)col * S + e] : 0.0;
            residual[(size_t)row * S + e] += values[(size_t)k * S + e] * (g - uc);
            values[(size_t)k * S + e] = 0.0;
          }
        }
      }
    }
  }
}

/* ------------------------------------------------------------------------ */
/* proj/include/enprop/kernels.hpp:15-26: sum = 0; sum += a_k * x_col in entry order */
void or_spmv(int S, int rows, const int* row_map, const int* col_entry, const double* values,
             const double* x, double* z) {
  for (int row = 0; row < rows; ++row)
    for (int e = 0; e < S; ++e) {
      double sum = 0.0;
      for (int k = row_map[row]; k < row_map[row + 1]; ++k)
        sum += values[(size_t)k * S + e] * x[(size_t)col_entry[k] * S + e];
      z[(size_t)row * S + e] = sum;
    }
}

/* spmv_outer, proj/include/enprop/kernels.hpp:38-56: sample-major layout,
 * component e sweeps the shared graph against values[e*nnz ...]. */
void or_spmv_outer(int S, int rows, int cols, const int* row_map, const int* col_entry,
                   const double* values, const double* x, double* z) {
  const size_t nnz = (size_t)row_map[rows];
  for (int e = 0; e < S; ++e) {
    const double* ve = values + (size_t)e * nnz;
    const double* xe = x + (size_t)e * cols;
    for (int row = 0; row < rows; ++row) {
      double sum = 0.0;
      for (int k = row_map[row]; k < row_map[row + 1]; ++k) sum += ve[k] * xe[col_entry[k]];
      z[(size_t)e * rows + row] = sum;
    }
  }
}

/* Per-lane dot in one of two orders.
 * SERIAL: proj/include/enprop/kernels.hpp:66-67 — acc = 0; acc += u*v row by row.
 * CANONICAL (the product's fast order, documented in DESIGN.md §4):
 *   rows are cut into segments of seg_rows (for a mesh: one z-plane of nodes),
 *   each segment into tiles of tile_rows (power of two) aligned at the segment
 *   start, and the tiles into blocks of OR_BLOCK_TILES consecutive tiles.
 *   A tile's products are padded with +0.0 to tile_rows and folded by
 *   v[i] = v[i] + v[i + half] for half = tile_rows/2, ..., 1; a block's tile sums
 *   are padded with +0.0 to OR_BLOCK_TILES and folded the same way; the segment
 *   sum is 0.0 + block_0 + block_1 + ... and the lane total 0.0 + seg_0 + ... */
static double fold(double* t, int n) {
  for (int half = n / 2; half >= 1; half /= 2)
    for (int i = 0; i < half; ++i) t[i] = t[i] + t[i + half];
  return t[0];
}

void or_dot_lanes(int S, int64_t n, const double* u, const double* v, int mode, int tile_rows,
                  int seg_rows, double* lanes) {
  if (mode == OR_DOT_SERIAL) {
    for (int e = 0; e < S; ++e) lanes[e] = 0.0;
    for (int64_t row = 0; row < n; ++row)
      for (int e = 0; e < S; ++e) lanes[e] += u[row * S + e] * v[row * S + e];
    return;
  }
  double* t = (double*)malloc(sizeof(double) * (size_t)tile_rows);
  double blk[OR_BLOCK_TILES];
  const int64_t block_rows = (int64_t)tile_rows * OR_BLOCK_TILES;
  for (int e = 0; e < S; ++e) {
    double total = 0.0;
    for (int64_t r0 = 0; r0 < n; r0 += seg_rows) {
      const int64_t r1 = r0 + seg_rows < n ? r0 + seg_rows : n;
      double seg = 0.0;
      for (int64_t b0 = r0; b0 < r1; b0 += block_rows) {
        for (int k = 0; k < OR_BLOCK_TILES; ++k) {
          const int64_t t0 = b0 + (int64_t)k * tile_rows;
          for (int i = 0; i < tile_rows; ++i) {
            const int64_t row = t0 + i;
            t[i] = row < r1 ? u[row * S + e] * v[row * S + e] : 0.0;
          }
          blk[k] = t0 < r1 ? fold(t, tile_rows) : 0.0;
        }
        seg = seg + fold(blk, OR_BLOCK_TILES);
      }
      total = total + seg;
    }
    lanes[e] = total;
  }
  free(t);
}

double or_dot(int S, int64_t n, const double* u, const double* v, int mode, int tile_rows,
              int seg_rows) {
  double lanes[64];
  double* l = S <= 64 ? lanes : (double*)malloc(sizeof(double) * (size_t)S);
  or_dot_lanes(S, n, u, v, mode, tile_rows, seg_rows, l);
  double acc = 0.0; /* ensemble.hpp:240-244 */
  for (int e = 0; e < S; ++e) acc += l[e];
  if (l != lanes) free(l);
  return acc;
}

/* proj/include/enprop/kernels.hpp:78-85: y = alpha*x + beta*y */
void or_axpby(int S, int64_t n, int per_lane, const double* alpha, const double* x,
              const double* beta, double* y) {
  for (int64_t row = 0; row < n; ++row)
    for (int e = 0; e < S; ++e) {
      const double a = per_lane ? alpha[e] : alpha[0];
      const double b = per_lane ? beta[e] : beta[0];
      y[row * S + e] = a * x[row * S + e] + b * y[row * S + e];
    }
}

/* ------------------------------------------------------------------------ */
/* proj/include/enprop/pcg.hpp:52-103, IdentityPreconditioner (:40-45).
 * Scalar solve on lane `lane` of [rows][S] storage = pcg_solve<double> on the
 * extracted component (kernels.hpp:125-160). */
static int pcg_lane(int S, int lane, int dot_mode, int T, int P, int rows, const int* row_map,
                    const int* col_entry, const double* values, const double* b, double tol,
                    int maxit, double* x, int* iterations, double* history, int hist_stride,
                    int* hist_len) {
  double* r = (double*)malloc(sizeof(double) * (size_t)rows);
  double* p = (double*)malloc(sizeof(double) * (size_t)rows);
  double* q = (double*)malloc(sizeof(double) * (size_t)rows);
  double* xs = (double*)calloc((size_t)rows, sizeof(double));
  double* bl = (double*)malloc(sizeof(double) * (size_t)rows);
  int status = OR_OK;
  for (int i = 0; i < rows; ++i) bl[i] = b[(size_t)i * S + lane];
  *hist_len = 0;
  *iterations = 0;
  const double b_norm = sqrt(or_dot(1, rows, bl, bl, dot_mode, T, P));
  if (b_norm == 0.0) {
    history[0] = 0.0;
    *hist_len = 1;
    goto done;
  }
  memcpy(r, bl, sizeof(double) * (size_t)rows);
  memcpy(p, r, sizeof(double) * (size_t)rows);
  double rz = or_dot(1, rows, r, r, dot_mode, T, P);
  for (int it = 0;; ++it) {
    const double relative = sqrt(or_dot(1, rows, r, r, dot_mode, T, P)) / b_norm;
    history[(size_t)(*hist_len) * hist_stride] = relative;
    ++*hist_len;
    if (relative < tol) {
      *iterations = it;
      break;
    }
    if (it >= maxit) {
      *iterations = it;
      status = OR_NO_CONVERGENCE;
      break;
    }
    /* spmv on the lane's values */
    for (int row = 0; row < rows; ++row) {
      double sum = 0.0;
      for (int k = row_map[row]; k < row_map[row + 1]; ++k)
        sum += values[(size_t)k * S + lane] * p[col_entry[k]];
      q[row] = sum;
    }
    const double pq = or_dot(1, rows, p, q, dot_mode, T, P);
    if (pq <= 0.0) {
      *iterations = it;
      status = OR_INDEFINITE;
      break;
    }
    const double alpha = rz / pq;
    const double one = 1.0, malpha = -alpha;
    or_axpby(1, rows, 0, &alpha, p, &one, xs);
    or_axpby(1, rows, 0, &malpha, q, &one, r);
    const double rz_next = or_dot(1, rows, r, r, dot_mode, T, P);
    const double beta = rz_next / rz;
    rz = rz_next;
    or_axpby(1, rows, 0, &one, r, &beta, p);
  }
done:
  for (int i = 0; i < rows; ++i) x[(size_t)i * S + lane] = xs[i];
  free(r); free(p); free(q); free(xs); free(bl);
  return status;
}

/* Coupled ensemble solve: pcg_solve<Ensemble<S>> (pcg.hpp:52-103) with the
 * coupled dot/norm2 of kernels.hpp:62-74 and scalar axpby coefficients. */
static int pcg_coupled(int S, int dot_mode, int T, int P, int rows, const int* row_map,
                       const int* col_entry, const double* values, const double* b, double tol,
                       int maxit, double* x, int* iterations, double* history, int* hist_len) {
  const size_t len = (size_t)rows * S;
  double* r = (double*)malloc(sizeof(double) * len);
  double* p = (double*)malloc(sizeof(double) * len);
  double* q = (double*)malloc(sizeof(double) * len);
  int status = OR_OK;
  memset(x, 0, sizeof(double) * len);
  *hist_len = 0;
  *iterations = 0;
  const double b_norm = sqrt(or_dot(S, rows, b, b, dot_mode, T, P));
  if (b_norm == 0.0) {
    history[0] = 0.0;
    *hist_len = 1;
    goto done;
  }
  memcpy(r, b, sizeof(double) * len);
  memcpy(p, r, sizeof(double) * len);
  double rz = or_dot(S, rows, r, r, dot_mode, T, P);
  for (int it = 0;; ++it) {
    const double relative = sqrt(or_dot(S, rows, r, r, dot_mode, T, P)) / b_norm;
    history[(*hist_len)++] = relative;
    if (relative < tol) {
      *iterations = it;
      break;
    }
    if (it >= maxit) {
      *iterations = it;
      status = OR_NO_CONVERGENCE;
      break;
    }
    or_spmv(S, rows, row_map, col_entry, values, p, q);
    const double pq = or_dot(S, rows, p, q, dot_mode, T, P);
    if (pq <= 0.0) {
      *iterations = it;
      status = OR_INDEFINITE;
      break;
    }
    const double alpha = rz / pq;
    const double one = 1.0, malpha = -alpha;
    or_axpby(S, rows, 0, &alpha, p, &one, x);
    or_axpby(S, rows, 0, &malpha, q, &one, r);
    const double rz_next = or_dot(S, rows, r, r, dot_mode, T, P);
    const double beta = rz_next / rz;
    rz = rz_next;
    or_axpby(S, rows, 0, &one, r, &beta, p);
  }
done:
  free(r); free(p); free(q);
  return status;
}

int or_pcg(int S, int flavour, int dot_mode, int tile_rows, int seg_rows, int rows,
           const int* row_map, const int* col_entry, const double* values, const double* b,
           double tol, int maxit, double* x, int* iterations, double* history, int* hist_len,
           int* lane_status) {
  if (S < 1 || rows < 0 || maxit < 0) return OR_INVALID;
  if (dot_mode == OR_DOT_CANONICAL &&
      (tile_rows < 1 || (tile_rows & (tile_rows - 1)) != 0 || seg_rows < 1))
    return OR_INVALID;
  if (flavour == OR_CG_COUPLED) {
    int st = pcg_coupled(S, dot_mode, tile_rows, seg_rows, rows, row_map, col_entry, values, b,
                         tol, maxit, x, iterations, history, hist_len);
    if (lane_status)
      for (int e = 0; e < S; ++e) lane_status[e] = st;
    return st;
  }
  int worst = OR_OK;
  for (size_t i = 0; i < (size_t)(maxit + 1) * S; ++i) history[i] = NAN;
  for (int e = 0; e < S; ++e) {
    int st = pcg_lane(S, e, dot_mode, tile_rows, seg_rows, rows, row_map, col_entry, values, b,
                      tol, maxit, x, &iterations[e], history + e, S, &hist_len[e]);
    if (lane_status) lane_status[e] = st;
    if (st > worst) worst = st;
  }
  return worst;
}
