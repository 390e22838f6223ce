/* enprop_b200 — C ABI of the B200-native ensemble hot path
 * (ensemble FEM assembly -> ensemble CRS SpMV -> ensemble CG) of
 * arXiv 1511.03703, drop-in for the reference library "enprop"
 * (/root/reference/proj/include/enprop).
 *
 * Conventions
 *  - Ensemble width s in {1,2,4,8,16,32} (the reference's compiled set,
 *    proj/src/bench.cpp:447-460).
 *  - Layouts are the reference's: values [nnz][s] fp64 (Ensemble<S> is a POD of
 *    S doubles, ensemble.hpp:105-106), vectors [rows][s] fp64, int32 row_map /
 *    col_entry (crs.hpp:19-69).  Device pointers unless a name says "host".
 *  - Calls are ordered on the context's stream.  Functions that return values
 *    to the host synchronise the stream.
 *  - Arithmetic is the reference's: fp64, no FMA contraction, left-to-right
 *    (proj/CMakeLists.txt:14 builds with -ffp-contract=off).  Assembly,
 *    Dirichlet, SpMV and axpby are bitwise equal to the reference.  Dot products
 *    and CG take a reduction order: ENPROP_DOT_SERIAL reproduces the reference
 *    bitwise (kernels.hpp:62-69); ENPROP_DOT_CANONICAL is the fast fixed tree of
 *    DESIGN.md §4 (bitwise equal to oracle/enprop_oracle.c's restatement).
 *  - Status codes mirror the reference's exceptions: ENPROP_ERR_INVALID for
 *    std::invalid_argument (e.g. kernels.hpp:17-18), NO_CONVERGENCE and
 *    INDEFINITE for SolverError (pcg.hpp:82-92).  enprop_last_error() holds
 *    the message (thread-local).
 */
#ifndef ENPROP_B200_H
#define ENPROP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENPROP_ABI_VERSION 1

enum {
  ENPROP_OK = 0,
  ENPROP_ERR_INVALID = 1,        /* std::invalid_argument in the reference */
  ENPROP_ERR_NO_CONVERGENCE = 2, /* SolverError: maxit reached (pcg.hpp:82-85) */
  ENPROP_ERR_INDEFINITE = 3,     /* SolverError: p'Ap <= 0 (pcg.hpp:88-92) */
  ENPROP_ERR_CUDA = 4,
  ENPROP_ERR_OOM = 5
};

enum { ENPROP_DOT_SERIAL = 0, ENPROP_DOT_CANONICAL = 1 };
enum { ENPROP_CG_COUPLED = 0, ENPROP_CG_UNCOUPLED = 1 };

/* Rows per canonical reduction tile. */
#define ENPROP_TILE_ROWS 16
/* Tiles per canonical reduction block. */
#define ENPROP_BLOCK_TILES 16

const char* enprop_last_error(void);
int enprop_abi_version(void);

/* ---------------------------------------------------------------- context */
typedef struct enprop_ctx enprop_ctx;
int enprop_ctx_create(int device, enprop_ctx** out);
int enprop_ctx_destroy(enprop_ctx* ctx);
/* cudaStream_t as void*; NULL selects the legacy default stream (torch's
 * default).  A new context runs on its own non-blocking stream. */
int enprop_ctx_set_stream(enprop_ctx* ctx, void* stream);
void* enprop_ctx_stream(enprop_ctx* ctx);
int enprop_ctx_synchronize(enprop_ctx* ctx);
/* number of enprop kernels launched through this context so far */
int64_t enprop_ctx_launch_count(enprop_ctx* ctx);
/* Tuning options (results are bitwise identical either way):
 *   ENPROP_OPT_FUSED_DIRECTION (default 0): 1 = form p = r + beta p inside the CG
 *   SpMV from gathers of r and p_old; 0 = separate direction pass, then an
 *   SpMV with a single gather.
 *   ENPROP_OPT_SYMMETRIC_STORAGE (default 1): problems created afterwards store
 *   only the diagonal + upper triangle of the (exactly symmetric) assembled
 *   operator and read each lower entry from its transposed slot
 *   (enprop_problem_expand_values rebuilds the full [nnz][s] values):
 *   1 = from s = 4 up (at s = 1, 2 the slot map costs what it saves), 2 = at
 *   every width, 0 = never (advection, alpha != 0, always stores all).
 *   ENPROP_OPT_SPMV_PIPELINE (default 0): 1 = enprop_spmv loads the next batch's
 *   column indices one batch ahead (software pipelining).
 *   ENPROP_OPT_SPMV_VARIANT (default -1 = auto): CG SpMV schedule
 *   (entries per gather batch / CTAs per SM): 0: 4/4, 1: 4/4 + index prefetch,
 *   2: 8/2, 3: 8/2 + index prefetch, 4: 4/4 zero-padded, 5: 8/3, 6: 16/1;
 *   auto = 2 with symmetric storage, 0 otherwise.
 *   ENPROP_OPT_GRAPHS (default 1; the environment variable ENPROP_GRAPHS=0
 *   makes it 0 for new contexts): CG iterations are replayed from a CUDA graph
 *   of one convergence-check chunk (check_every iterations) instead of being
 *   launched kernel by kernel (not while profiling).
 * Options are per context: calls through a context (and through problems and
 * slab solvers created on it) launch with that context's settings only. */
/*   ENPROP_OPT_PDL (default 0): launch the CG loop's kernels with
 *   programmatic dependent launch (the next kernel is scheduled while the
 *   previous one drains; it waits for its completion before reading).
 *   Measured: +2-4% on single-stream s = 4 / 16 solves, -1% with three
 *   concurrent s = 32 groups (early-scheduled CTAs hold SMs other streams
 *   could use). */
enum {
  ENPROP_OPT_FUSED_DIRECTION = 1,
  ENPROP_OPT_SPMV_PIPELINE = 2,
  ENPROP_OPT_SYMMETRIC_STORAGE = 3,
  ENPROP_OPT_SPMV_VARIANT = 5,
  ENPROP_OPT_PDL = 6,
  ENPROP_OPT_GRAPHS = 7
};
int enprop_ctx_set_option(enprop_ctx* ctx, int option, int value);
/* Event timing of the CG SpMV kernel launches on the context stream (used by
 * bench.py for the roofline). Returns the totals accumulated since the last
 * reset; enable = 1/0 turns timing on/off and resets, enable = -1 only reads. */
int enprop_ctx_profile(enprop_ctx* ctx, int enable, double* spmv_ms, int64_t* spmv_launches);
/* Per-phase totals of the profiled CG iterations, ms[11]: [0] SpMV phase
 * (direction + SpMV), [1] PQ finalize, [2] update, [3] RR finalize, [4] whole
 * working iterations; per profiled solve: [5] whole solve on the GPU, [6] setup
 * and initial residual, [7] iteration loop (incl. early-exit iterations),
 * [8] iterations enqueued past convergence (early-exit); per iteration again:
 * [9] direction pass, [10] SpMV kernel. */
int enprop_ctx_profile_detail(enprop_ctx* ctx, double* ms, int64_t* iterations);

int enprop_malloc(enprop_ctx* ctx, size_t bytes, void** dptr);
int enprop_free(enprop_ctx* ctx, void* dptr);
/* stream-ordered copies; both return after the copy completed */
int enprop_memcpy_h2d(enprop_ctx* ctx, void* dst, const void* host_src, size_t bytes);
int enprop_memcpy_d2h(enprop_ctx* ctx, void* host_dst, const void* src, size_t bytes);

/* ------------------------------------------------------- problem parameters */
/* KlField(num_terms, mean, sigma, correlation_length)  (kl.hpp:39-95) */
typedef struct {
  int num_terms;
  double mean, sigma, correlation_length;
} enprop_kl_params;

/* PdeCoefficients (fem.hpp:21-25) */
typedef struct {
  double alpha, beta;
  double velocity[3];
} enprop_pde_coeffs;

/* DirichletBc (fem.hpp:29-32) */
typedef struct {
  double x0_value, x1_value;
} enprop_dirichlet_bc;

/* ------------------------------------------------------------ mesh & field */
/* (3(n+1)-2)^3 stored entries of the 27-point node graph (mesh.cpp:13-55) */
int64_t enprop_mesh_nnz(int cells_per_axis);
/* build_node_graph(StructuredMesh(n)) into device arrays, bit-exact
 * (mesh.cpp:13-55). row_map[(n+1)^3 + 1], col_entry[enprop_mesh_nnz(n)]. */
int enprop_build_node_graph(enprop_ctx* ctx, int cells_per_axis, int* row_map, int* col_entry);
/* KlField eigen-structure on the host (kl.cpp:41-89): per retained mode i
 * mode_axes[3i..3i+2], mode_eigenvalue[i]; per axis mode t axis_frequency[t],
 * axis_eigenvalue[t], axis_inverse_norm[t], axis_cosine[t]. Arrays of num_terms. */
int enprop_kl_describe(const enprop_kl_params* kl, int* mode_axes, double* mode_eigenvalue,
                       double* axis_frequency, double* axis_eigenvalue,
                       double* axis_inverse_norm, int* axis_cosine);

/* ---------------------------------------------------------------- samples */
/* draw_samples (samples.cpp:7-18): out[count][num_terms], coordinate j of
 * sample i = (mt19937_64(seed) >> 11) * 2^-52 - 1 in draw order, uniform in
 * [-1, 1); bitwise the reference's sequence. INVALID for num_terms < 1 or
 * count < 0. Host memory. */
int enprop_draw_samples(uint64_t seed, int count, int num_terms, double* out);
/* pack_sample_group<S> (samples.hpp:18-31): out[j][e] = samples[group_start +
 * e][j] for j < num_terms, e < s -- the [num_terms][s] y layout of
 * enprop_assemble / enprop_problem_assemble. samples is [count][num_terms].
 * INVALID when the group runs past count (the reference's "not enough samples
 * for the group"). Host memory. */
int enprop_pack_sample_group(const double* samples, int count, int num_terms, int group_start,
                             int s, double* out);

/* ----------------------------------------------------------------- kernels */
/* assemble<Ensemble<s>> (fem.hpp:115-202) of the unit-cube diffusion problem
 * on the n^3 hex mesh; optionally followed by apply_dirichlet (fem.hpp:218-243)
 * fused in the same kernel when bc != NULL.
 *   u        [rows][s] current iterate, NULL means all zeros
 *   y        [num_terms][s] sample coordinates (pack_sample_group layout)
 *   row_map  graph from enprop_build_node_graph
 *   values   [nnz][s] out; residual [rows][s] out (both overwritten) */
int enprop_assemble(enprop_ctx* ctx, int s, int cells_per_axis, const enprop_kl_params* kl,
                    const enprop_pde_coeffs* coeffs, const double* u, const double* y,
                    const int* row_map, double* values, double* residual,
                    const enprop_dirichlet_bc* bc);
/* apply_dirichlet (fem.hpp:218-243) on an assembled mesh system, in place. */
int enprop_apply_dirichlet(enprop_ctx* ctx, int s, int cells_per_axis,
                           const enprop_dirichlet_bc* bc, const int* row_map,
                           const int* col_entry, const double* u, double* values,
                           double* residual);

/* spmv (kernels.hpp:15-26): z = A x, general CRS, bitwise equal per lane. */
int enprop_spmv(enprop_ctx* ctx, int s, int num_rows, int num_cols, const int* row_map,
                const int* col_entry, const double* values, const double* x, double* z);

/* spmv_outer (kernels.hpp:38-56) on the sample-major layout of
 * OuterEnsembleMatrix (crs.hpp:138-147): values[e*nnz + k], x[e*num_cols + c],
 * z[e*num_rows + row] for e < ensemble_size; any ensemble_size >= 1. Each
 * component is bitwise the reference's scalar product. (Device pointers.) */
int enprop_spmv_outer(enprop_ctx* ctx, int ensemble_size, int num_rows, int num_cols, int64_t nnz,
                      const int* row_map, const int* col_entry, const double* values,
                      const double* x, double* z);

/* Diagnostics: the narrow-ensemble SpMV configuration enprop_spmv launches
 * for width s (CTA threads, register cap -- 0 = uncapped -- and staging mode;
 * set by the ENPROP_SMALL_* environment switches), and whether s is routed to
 * it at all (s <= ENPROP_SMALL_MAX). */
int enprop_spmv_small_config(int s, int* routed, int* threads, int* reg_cap, int* stage_mode);

/* dot (kernels.hpp:62-69): per-lane sums lanes_host[s] (may be NULL) and the
 * coupled reduce_sum coupled_host (may be NULL) in the given order.
 * seg_rows is the canonical segment length (ignored for SERIAL). */
int enprop_dot(enprop_ctx* ctx, int s, int64_t n, const double* u, const double* v,
               int dot_mode, int seg_rows, double* lanes_host, double* coupled_host);

/* axpby (kernels.hpp:78-85): y = alpha*x + beta*y. per_lane != 0: alpha/beta
 * are s host doubles (Ensemble coefficients), else one host double each. */
int enprop_axpby(enprop_ctx* ctx, int s, int64_t n, int per_lane, const double* alpha_host,
                 const double* x, const double* beta_host, double* y);

/* ----------------------------------------------------------------------- CG */
/* Identity-preconditioned CG from x0 = 0 (pcg.hpp:52-103).
 *   COUPLED   = pcg_solve<Ensemble<s>>: one coupled norm/decision.
 *   UNCOUPLED = s x pcg_solve<double> on extracted components
 *               (bench.cpp:340-349): per-lane alpha, beta and stopping.
 * Outputs (host): iterations[lanes], lane_status[lanes], history
 * [(maxit+1)][lanes] relative residuals (NaN past a lane's end),
 * hist_len[lanes]; lanes = 1 (COUPLED) or s (UNCOUPLED).  Any may be NULL.
 * Returns the worst status over lanes. */
typedef struct {
  int flavour;   /* ENPROP_CG_* */
  int dot_mode;  /* ENPROP_DOT_* */
  int seg_rows;  /* canonical segment (a mesh z-plane: (n+1)^2); <=0 -> 4096 */
  double tol;
  int max_iterations;
  int check_every; /* host polls convergence every k iterations (<=0 -> 16) */
} enprop_cg_options;

int enprop_cg(enprop_ctx* ctx, int s, int num_rows, const int* row_map, const int* col_entry,
              const double* values, const double* b, double* x, const enprop_cg_options* opt,
              int* iterations, int* lane_status, double* history, int* hist_len);

/* -------------------------------------------------- device-resident problem */
/* The performance path: graph, KL tables, matrix and CG workspaces stay in HBM;
 * one call assembles + imposes Dirichlet + solves A x = -residual for one
 * sample group (bench.cpp:286-299 with IdentityPreconditioner). */
typedef struct {
  int cells_per_axis;
  int ensemble_size;
  enprop_kl_params kl;
  enprop_pde_coeffs coeffs;
  enprop_dirichlet_bc bc;
} enprop_problem_desc;

typedef struct enprop_problem enprop_problem;
int enprop_problem_create(enprop_ctx* ctx, const enprop_problem_desc* desc, enprop_problem** out);
int enprop_problem_destroy(enprop_problem* p);
/* device views (owned by the problem) */
int enprop_problem_views(enprop_problem* p, int* num_rows, int64_t* nnz, const int** row_map,
                         const int** col_entry, double** values, double** residual,
                         double** solution);
/* stored value entries (nnz, or (nnz + rows)/2 with symmetric storage) and the
 * entry -> slot map (NULL for full storage); `values` of enprop_problem_views is
 * the stored array */
int enprop_problem_storage(enprop_problem* p, int64_t* nnz_stored, const int** vpos);
/* full [nnz][s] values of the assembled operator into a device buffer */
int enprop_problem_expand_values(enprop_problem* p, double* values_full);
/* assemble + Dirichlet from device samples y [num_terms][s] (u = 0) */
int enprop_problem_assemble(enprop_problem* p, const double* y);
/* CG on the assembled system with rhs = -residual; solution in the problem */
int enprop_problem_solve(enprop_problem* p, const enprop_cg_options* opt, int* iterations,
                         int* lane_status, double* history, int* hist_len);
/* End to end from HOST buffers: y_host [num_terms][s] -> x_host [rows][s]. */
int enprop_problem_solve_host(enprop_problem* p, const double* y_host, double* x_host,
                              const enprop_cg_options* opt, int* iterations, int* lane_status);

/* NewtonOptions (fem.hpp:244-249) without the multigrid block: the linear
 * solves use the identity preconditioner (IdentityPreconditioner, pcg.hpp:40-46). */
typedef struct {
  double tol;          /* on the coupled residual norm, relative to the first (default 1e-8) */
  int max_iterations;  /* Newton steps (default 20) */
  enprop_cg_options linear;
} enprop_newton_options;

/* newton_solve (fem.hpp:265-302) on the device-resident problem: from u = 0,
 * assemble residual and Jacobian at u (nonlinear terms of the problem's
 * PdeCoefficients), impose Dirichlet, stop when the coupled residual norm is
 * below tol x the first (or the first is 0), else solve J du = -f by CG and
 * u = 1.0*du + 1.0*u (axpby). y: device [num_terms][s]. The converged iterate is
 * left in the problem's `solution` view. residual_norms (host, may be NULL,
 * max_iterations + 1 entries) receives the norm before each step, num_norms
 * their count; total_cg_iterations sums each linear solve's iterations (the
 * maximum over lanes for uncoupled solves). Errors: NO_CONVERGENCE after
 * max_iterations steps (norms filled), or the linear solver's failure. */
int enprop_problem_newton(enprop_problem* p, const double* y, const enprop_newton_options* opt,
                          int* newton_iterations, int* total_cg_iterations,
                          double* residual_norms, int* num_norms);

/* ------------------------------------------- multigrid preconditioner (f4) */
/* MgOptions (multigrid.hpp:14-20); NULL options select the defaults
 * {500, 2, 30.0, 1.1, 40}. */
typedef struct {
  int coarse_row_threshold;
  int chebyshev_degree;
  double eigenvalue_ratio;
  double eigenvalue_boost;
  int power_iterations;
} enprop_mg_options;

typedef struct enprop_mg enprop_mg;
/* build_hierarchy (multigrid.hpp:362-396) of the ensemble operator values
 * [nnz][s] (device CRS, full storage): aggregation, Galerkin products and
 * power-iteration eigenvalue estimates on the host in the reference's order,
 * the coarsest level's dense LU per component on the device (bitwise the
 * reference's factors). The hierarchy owns copies of every level. */
int enprop_mg_build(enprop_ctx* ctx, int s, int num_rows, const int* row_map, const int* col_entry,
                    const double* values, const enprop_mg_options* opt, enprop_mg** out);
int enprop_mg_destroy(enprop_mg* h);
/* levels, rows per level (<= max_levels entries) and the smoothed levels'
 * lambda_max estimates [num_levels-1][s] (each may be NULL) */
int enprop_mg_describe(enprop_mg* h, int* num_levels, int* rows, int max_levels, double* lambda_max);
/* one V-cycle (multigrid.hpp:402-425) on the finest level: x updated in place
 * toward A x = b (device [rows][s]); MgPreconditioner = one V-cycle from x = 0 */
int enprop_mg_vcycle(enprop_mg* h, const double* b, double* x);
/* pcg_solve(A, b, MgPreconditioner(h), cfg) (pcg.hpp:52-103) from x0 = 0, in
 * the reference's serial dot order: COUPLED = pcg_solve<Ensemble<s>>,
 * UNCOUPLED = s x pcg_solve<double> (per-lane scalars; converged lanes frozen).
 * Outputs as enprop_cg. */
int enprop_mg_pcg(enprop_mg* h, const double* b, double* x, const enprop_cg_options* opt,
                  int* iterations, int* lane_status, double* history, int* hist_len);

/* newton_solve (fem.hpp:265-302) exactly as the reference runs it: every
 * linear solve is pcg_solve(J, -f, MgPreconditioner(build_hierarchy(J, mg)))
 * (mg NULL = MgOptions defaults), serial dot order. Same outputs as
 * enprop_problem_newton. */
int enprop_problem_newton_mg(enprop_problem* p, const double* y, const enprop_newton_options* opt,
                             const enprop_mg_options* mg, int* newton_iterations,
                             int* total_cg_iterations, double* residual_norms, int* num_norms);

/* ------------------------------------ multi-GPU: slab domain decomposition */
/* The node planes z = k of the mesh are split over nranks like the
 * reference's partition (partition.cpp:31-72; lower ranks take the extra
 * plane). Each rank assembles its own rows (no communication), and each CG
 * iteration exchanges one ghost plane with each neighbour (halo of p) and
 * all-gathers the per-plane dot sums; totals are formed in global plane order
 * (the canonical order), so results are bitwise independent of nranks.
 *   nccl_id != NULL: this process is `rank` of an NCCL job, one GPU per rank
 *                    (id from enprop_nccl_unique_id on rank 0, broadcast by the host);
 *   nccl_id == NULL: all nranks are emulated in this process on ctx's GPU with
 *                    stream-ordered device copies as transport (testing). */
int enprop_nccl_unique_id(void* out, size_t bytes);
typedef struct enprop_dist enprop_dist;
int enprop_dist_create(enprop_ctx* ctx, const enprop_problem_desc* desc, int nranks, int rank,
                       const void* nccl_id, enprop_dist** out);
/* The same over the CUDA-IPC transport: one process per rank on any GPUs of
 * one node -- several ranks may share one GPU, which NCCL refuses. `job` names
 * the host board (/dev/shm/enprop_b200_<job>) that every rank of the job opens;
 * it must be unique per job (e.g. a random token from rank 0). Peers exchange
 * through their exported buffers and interprocess events: stream waits and
 * cudaMemcpyAsync (NVLink P2P between GPUs), never a kernel waiting on another
 * rank. Blocks until all nranks have joined (ENPROP_ERR_CUDA after 120 s). */
int enprop_dist_create_ipc(enprop_ctx* ctx, const enprop_problem_desc* desc, int nranks, int rank,
                           const char* job, enprop_dist** out);
int enprop_dist_destroy(enprop_dist* d);
/* assemble + Dirichlet of every local rank's rows; y [num_terms][s] on the device */
int enprop_dist_assemble(enprop_dist* d, const double* y);
/* CG on A x = -residual, canonical dot order (DOT_SERIAL is INVALID here) */
int enprop_dist_solve(enprop_dist* d, const enprop_cg_options* opt, int* iterations,
                      int* lane_status);
/* newton_solve (fem.hpp:265-302) over the slabs, with Alg. 2's halo step: from
 * u = 0, every step imports the neighbours' boundary planes of u, assembles
 * the local rows at u, forms the coupled residual norm in the canonical order,
 * and solves J du = -f by enprop_dist_solve (identity preconditioner). Every
 * rank takes the same decisions; norms, steps, CG iterations and u are bitwise
 * those of enprop_problem_newton on one GPU with DOT_CANONICAL. The iterate
 * ends in each local rank's x (enprop_dist_local). Outputs and errors as
 * enprop_problem_newton; linear.dot_mode must be DOT_CANONICAL. */
int enprop_dist_newton(enprop_dist* d, const double* y, const enprop_newton_options* opt,
                       int* newton_iterations, int* total_cg_iterations, double* residual_norms,
                       int* num_norms);
/* Staged slabs (s in {4, 16, 32}): the local rank's SpMV stages and how many
 * of them are interior (rows at least one plane from every ghost plane). Each
 * CG iteration runs the interior stages while the halo is in flight and the
 * rest after it. Unstaged slabs report 0 / 0. */
int enprop_dist_stages(enprop_dist* d, int index, int* interior, int* total);
/* local ranks (1 with NCCL, nranks when emulated) and their owned rows / solution */
int enprop_dist_local_count(enprop_dist* d);
int enprop_dist_local(enprop_dist* d, int index, int* rank, int* row_begin, int* rows,
                      double** x);
/* Measured halo exchange (the solver's own exchange of one p buffer: one plane
 * of s values to each neighbour, NCCL or the emulated device copies), mean
 * seconds per exchange over `reps`, CUDA events on the context's stream. */
int enprop_dist_time_halo(enprop_dist* d, int reps, double* seconds);

/* One message of a halo exchange (ExchangeRecord, halo.hpp:86-91): here `time`
 * is MEASURED -- the sender's cumulative seconds of its messages in this
 * exchange (CUDA events around each copy / NCCL send-receive), where the
 * reference accumulates a virtual clock. */
typedef struct {
  int rank, neighbor;
  int64_t bytes;
  double time;
} enprop_exchange_record;
/* One measured halo exchange of the solver's p buffer (one plane of s values
 * to each neighbour), records in the reference's order (sender rank, then its
 * lower link before its upper link: partition.cpp:59-72). Emulated: every
 * rank's messages; NCCL / IPC: the messages this process takes part in (IPC
 * pulls: sender = the neighbour). elapsed = max cumulative time over senders. */
int enprop_dist_exchange_trace(enprop_dist* d, enprop_exchange_record* out, int max_records,
                               int* count, double* elapsed_seconds);

/* ------------------------------------------------ halo timing model (host) */
/* write_exchange_trace_csv (halo.cpp:192-202): header
 * "rank,neighbor,bytes,virtual_time", one "%d,%d,%lld,%.17g" line per record;
 * INVALID when the file cannot be written. */
int enprop_write_exchange_trace_csv(const char* path, const enprop_exchange_record* recs, int count);
/* fit_halo_model (halo.cpp:156-181): least-squares T(s) = a + b*s through
 * (s[i], t[i]), i < n; INVALID for n < 2 or all s equal (singular). */
int enprop_fit_halo_model(int n, const double* s, const double* t, double* a, double* b,
                          double* residual_sum_of_squares);
/* predicted_speedup (halo.cpp:183-188): s*(a + b)/(a + b*s); INVALID for s < 1
 * or a zero exchange time. */
int enprop_predicted_speedup(double a, double b, double s, double* speedup);

#ifdef __cplusplus
}
#endif
#endif /* ENPROP_B200_H */
