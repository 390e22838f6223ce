/* TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (proj/ of arxiv 1511.03703,
 * "enprop"): mesh graph, KL field, Q1 assembly, Dirichlet elimination, ensemble
 * SpMV, coupled/per-lane dots, axpby and identity-preconditioned CG.  It is the
 * checker for the CUDA path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  It is pinned bitwise against the unmodified
 * reference library (oracle/_ref, built by oracle/Makefile) in
 * tests/test_oracle.py and against golden vectors in tests/golden/.
 *
 * Layouts follow the reference: ensemble width S, values [nnz][S],
 * vectors [rows][S] (proj/include/enprop/ensemble.hpp:105-106).
 * Compile with -ffp-contract=off (proj/CMakeLists.txt:14): every expression is
 * written in the reference's left-to-right order with no contraction.
 */
#ifndef ENPROP_ORACLE_H
#define ENPROP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_TERMS 64
#define OR_BLOCK_TILES 16 /* canonical order: tiles per block */

typedef struct {
  int m;
  double mean, sigma, corr_length;
  /* axis eigenpairs t < m (kl.hpp:17-28) */
  double axis_freq[OR_MAX_TERMS], axis_eig[OR_MAX_TERMS], axis_invnorm[OR_MAX_TERMS];
  int axis_cos[OR_MAX_TERMS];
  /* retained 3D modes i < m (kl.cpp:64-89) */
  int mode_axes[OR_MAX_TERMS][3];
  double mode_eig[OR_MAX_TERMS], mode_sqrt_eig[OR_MAX_TERMS];
} or_kl_field;

/* dot-product reduction orders */
enum { OR_DOT_SERIAL = 0, OR_DOT_CANONICAL = 1 };
/* CG flavours */
enum { OR_CG_COUPLED = 0, OR_CG_UNCOUPLED = 1 };
/* status codes (shared with the product C ABI) */
enum { OR_OK = 0, OR_INVALID = 1, OR_NO_CONVERGENCE = 2, OR_INDEFINITE = 3 };

/* samples.cpp:7-18 */
void or_draw_samples(uint64_t seed, int count, int m, double* out /*[count][m]*/);
/* mesh.cpp:13-55; row_map[(n+1)^3+1], col_entry[(3n+1)^3] */
int64_t or_graph_nnz(int n);
void or_build_graph(int n, int* row_map, int* col_entry);
/* kl.cpp:41-89 */
int or_kl_init(or_kl_field* f, int m, double mean, double sigma, double corr_length);
/* kl.hpp:67-81 for one point; y [m][S], out [S] */
void or_kl_evaluate(const or_kl_field* f, int S, const double x[3], const double* y, double* out);

/* fem.hpp:115-202 (+ fem.hpp:218-243 when dirichlet != 0). u may be NULL (= 0). */
void or_assemble(int S, int n, const or_kl_field* f, double alpha, double beta,
                 const double velocity[3], const double* u, const double* y, int dirichlet,
                 double bc_x0, double bc_x1, double* values, double* residual);
/* fem.hpp:218-243 on an assembled system */
void or_apply_dirichlet(int S, int n, double bc_x0, double bc_x1, const int* row_map,
                        const int* col_entry, const double* u, double* values, double* residual);

/* kernels.hpp:15-26 */
void or_spmv(int S, int rows, const int* row_map, const int* col_entry, const double* values,
             const double* x, double* z);
/* kernels.hpp:38-56 (sample-major: values[e*nnz+k], x[e*cols+c], z[e*rows+row]) */
void or_spmv_outer(int S, int rows, int cols, const int* row_map, const int* col_entry,
                   const double* values, const double* x, double* z);
/* per-lane sums of u.v in the chosen order; kernels.hpp:62-69 for SERIAL */
void or_dot_lanes(int S, int64_t n, const double* u, const double* v, int mode, int tile_rows,
                  int seg_rows, double* lanes /*[S]*/);
/* coupled dot = reduce_sum over lanes (ensemble.hpp:237-244) */
double or_dot(int S, int64_t n, const double* u, const double* v, int mode, int tile_rows,
              int seg_rows);
/* kernels.hpp:78-85 */
void or_axpby(int S, int64_t n, int per_lane, const double* alpha, const double* x,
              const double* beta, double* y);

/* pcg.hpp:52-103 with IdentityPreconditioner (pcg.hpp:40-45).
 * COUPLED: one history/iteration count (iterations[0], history [maxit+1]).
 * UNCOUPLED: per-lane pcg_solve<double> semantics (bench.cpp:340-349):
 *   iterations[S], lane_status[S], history [maxit+1][S] (NaN past a lane's end),
 *   hist_len[S].  Return value: worst status over lanes. */
int or_pcg(int S, int flavour, int dot_mode, int tile_rows, int seg_rows, int rows,
           const int* row_map, const int* col_entry, const double* values, const double* b,
           double tol, int maxit, double* x, int* iterations, double* history, int* hist_len,
           int* lane_status);

#ifdef __cplusplus
}
#endif
#endif
