// Internal host-side interface of the enprop_b200 kernels (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ep_tilemap.h"

namespace ep {

// Device-resident per-problem assembly constants (fem.hpp:76-98, :133-191),
// all computed on the host in the reference's operation order.
struct AsmTables {
  double G[8][8][8];    // [q][i][j]: (gx_j*gx_i + gy_j*gy_i) + gz_j*gz_i, g* = gradient*grad_scale
  double ADV[8][8][8];  // [q][i][j]: advect_ij = (alpha*((vx*gx_j + vy*gy_j) + vz*gz_j))*n_i
  double NN[8][8][8];   // [q][i][j]: n_j*n_i
  double GS[8][8][3];   // [q][c][axis]: gradient*grad_scale
  double VAL[8][8];     // [q][c]: basis value
  double wd;            // (h/2)^3
  double alpha, beta, vx, vy, vz;
};

struct AsmArgs {
  int n;                 // cells per axis
  int rows;              // rows assembled by this launch ((n+1)^3 on one GPU)
  int row_begin;         // global node id of local row 0 (a rank's slab; 0 on one GPU)
  int u_shift;           // u is indexed by (global node - u_shift)
  int kc_lo;             // lowest cell plane read: a slab's lo ghost rows (only their
                         // upper slots toward the owned plane are used) skip the
                         // cells below, so u is read only inside the rank's halo
  int m;                 // KL terms
  double mean;           // kappa0
  const double* F;       // KL axis tables [m][2n]: f_t((c + off_b) * h)
  const AsmTables* tab;  // device copy (kept for the dist path's uploads)
  AsmTables T;           // the same tables by value: kernel-parameter (constant bank) reads
  const int* row_map;    // device
  const double* u;       // [rows][s] or nullptr (= 0)
  const double* y;       // [m][s]
  double* values;        // [nnz][s]
  double* residual;      // [rows][s]
  const int* vpos;       // symmetric storage: write only col >= row, at vpos[entry]
  int dirichlet;         // fuse apply_dirichlet
  int nonlinear;         // alpha != 0 || beta != 0
  double bc0, bc1;
  int mode_axes[64][3];
  double mode_sl[64];    // sigma * sqrt(lambda_i)
};

// CG state on the device (one per solve).  Coupled solves store their scalars
// replicated across lanes so the vector kernels are flavour-agnostic.
struct CgState {
  int it, done, status, flavour;
  int s, maxit, pad0, pad1;
  double tol;
  double rz[32], alpha[32], beta[32], bnorm[32];
  int active[32], iters[32], lane_status[32], hist_len[32];
  // lanes whose x += alpha*p of the last finished iteration is still owed:
  // x updates are deferred into the next direction pass (ep_kernels.cu)
  int pending[32];
};

enum Phase { kPhaseNone = 0, kPhaseInit = 1, kPhasePQ = 2, kPhaseRR = 3 };

// Fused canonical finalize (ep_kernels.cu tiles_finish): where the tile
// partials go, the self-resetting arrival counters, and what to do with the
// lane totals (a CG scalar phase, or write them to lanes_out for kPhaseNone).
// Counter words of one CG workspace (kCounterInts ints, zero at allocation;
// each kernel that uses one leaves it as it found it, except the barrier's
// monotonic generation): seg_done (finalize arrivals), the staged SpMV's grid
// barrier (count, generation) and its stage ticket (dynamic stage claims).
constexpr int kCounterInts = 4;

struct FinArgs {
  double* partials;  // [num_tiles][s]
  double* seg_sums;  // [num_segs][s]
  int* seg_done;     // [1] finalize arrivals, zero between launches
  int* bar;          // [2] grid barrier: arrivals (zero between launches), generation
  int* ticket;       // [1] staged SpMV stage claims, zero between launches
  double* prod;      // serial order: per-(row, sample) products p*q written by the SpMV
  int phase;
  CgState* cg;
  double* hist;
  double* lanes_out;  // [s + 1] for kPhaseNone
  int seg_only;       // multi-GPU: stop at the segment sums (seg_sums) — the
                      // total over all ranks' segments is k_fin_gathered's job
  int defer;          // producing kernels only write tile partials (always 1:
                      // launch_fin_segments forms the segment sums / total / phase)
};

cudaError_t launch_build_graph(int n, int* row_map, int* col_entry, cudaStream_t st);
// rows [row_begin, row_begin + rows) of the global node graph, entries
// renumbered from 0 and columns shifted by -col_shift (a rank's slab)
cudaError_t launch_build_graph_range(int n, int row_begin, int rows, int col_shift, int* row_map,
                                     int* col_entry, cudaStream_t st);
// deferred canonical finalize: one block per segment forms 0.0 + tile_0 + ... from
// f.partials; unless f.seg_only, the last block forms the total and runs f.phase
cudaError_t launch_fin_segments(int s, const TileMap& tm, const FinArgs& f, cudaStream_t st);
// multi-GPU finalize: total over all planes in global order from the
// all-gathered per-rank segment sums, gathered[plane_pos[k]][s], then `phase`
cudaError_t launch_fin_gathered(int s, int planes, const double* gathered, const int* plane_pos,
                                int phase, CgState* cg, double* hist, double* lanes_out,
                                cudaStream_t st);
cudaError_t launch_assemble(int s, const AsmArgs& a, cudaStream_t st);
cudaError_t launch_dirichlet(int s, int n, double bc0, double bc1, const int* row_map,
                             const int* col_entry, const double* u, double* values,
                             double* residual, cudaStream_t st);
cudaError_t launch_spmv(int s, int rows, const int* row_map, const int* col_entry,
                        const double* values, const double* x, double* z, bool pipe,
                        cudaStream_t st);
// narrow ensembles (s <= 16): row blocks staged in shared memory (ep_outer.cu)
int spmv_small_max();  // widest s routed to launch_spmv_small (16; 8 or 32 by env)
void spmv_small_config(int s, int* threads, int* reg_cap, int* stage_mode);
cudaError_t launch_spmv_small(int s, int rows, const int* row_map, const int* col_entry,
                              const double* values, const double* x, double* z, cudaStream_t st);
// spmv_outer (kernels.hpp:38-56): sample-major values[e*nnz + k], x[e*cols + c], z[e*rows + row]
cudaError_t launch_spmv_outer(int s, int rows, int cols, int64_t nnz, const int* row_map,
                              const int* col_entry, const double* values, const double* x,
                              double* z, cudaStream_t st);
cudaError_t launch_axpby(int s, int64_t n, int per_lane, const double* alpha, const double* beta,
                         const double* x, double* y, cudaStream_t st);
// canonical dot of u.v with the fused finalize running f.phase
cudaError_t launch_dot_tiles(int s, const TileMap& tm, const double* u, const double* v,
                             const FinArgs& f, cudaStream_t st);
// serial (reference-order) dot straight from the vectors, then f.phase; uses
// f.seg_sums[0..s) as the lane buffer and f.seg_done as its arrival counter
// (any alignment; the chain kernel below is the fast path)
cudaError_t launch_fin_serial(int s, int rows, const double* u, const double* v, const FinArgs& f,
                              cudaStream_t st);
// serial (reference-order) dot by one chain CTA (ep_chain.cu): lane e of its
// consumer warp runs sample e's chain acc = 0.0; acc += a_row (kernels.hpp:66-67)
// over rows staged through shared memory by bulk copies, then f.phase.
//   kChainGiven: a_row = u[row] (products already formed, v unused)
//   kChainSquare: a_row = u[row]*u[row];  kChainProduct: a_row = u[row]*v[row]
// u, v 16-byte aligned (chain_aligned); otherwise use launch_fin_serial.
enum ChainKind { kChainGiven = 0, kChainSquare = 1, kChainProduct = 2 };
bool chain_aligned(const void* u, const void* v);
cudaError_t launch_chain(int s, int rows, const double* u, const double* v, int kind,
                         const FinArgs& f, cudaStream_t st);
// q = A p_new with p_new = (it==0 ? r : r + beta*p_old) formed on the fly; writes
// p_new and q; with tiles, also the canonical p_new.q and its CG phase (f)
// fused_dir = false: a separate k_cg_direction pass writes p_new first and the
// SpMV gathers it directly (one gather per entry instead of two)
// the split direction pass alone (multi-GPU: the halo goes between it and the SpMV)
cudaError_t launch_cg_direction(int s, int rows, const double* r, const double* p_old,
                                double* p_new, double* x, const CgState* cg, cudaStream_t st);
// p_gather: base of the gathered p (the rank's ghost-extended layout; == p_new on
// one GPU). run_direction (split schedule): launch the direction pass first;
// false when the caller already ran it (multi-GPU: with the halo in between).
cudaError_t launch_cg_spmv(int s, bool tiles, bool fused_dir, bool run_direction,
                           const TileMap& tm, const int* row_map, const int* col_entry,
                           const double* values, const double* r, const double* p_old,
                           double* p_new, double* q, double* x, const double* p_gather,
                           const int* vpos, const FinArgs& f, cudaStream_t st);
// r -= alpha q on active lanes; with tiles, also r.r and its phase
cudaError_t launch_cg_update(int s, bool tiles, const TileMap& tm, double* r, const double* q,
                             const FinArgs& f, cudaStream_t st);
// Symmetric (diagonal + upper) value storage: vpos[nnz] maps each full-CRS entry
// to its stored slot; nnz_up = stored entries. Fails (InvalidValue) if the
// pattern is not structurally symmetric.
// up_start (optional, rows + 1 ints): first stored slot of each row.
// base: graph row r has coordinate r - base and columns are coordinates (a
// slab's store rows = `base` ghost rows + owned rows); ghost rows' lower
// entries get vpos = -1 (never read).
cudaError_t build_sym(int rows, const int* row_map, const int* col_entry, int* vpos,
                      int64_t* nnz_up, cudaStream_t st, int* up_start = nullptr, int base = 0);
// full[k] = up[vpos[k]] (views / checks)
cudaError_t launch_sym_expand(int s, int64_t nnz, const int* vpos, const double* up, double* full,
                              cudaStream_t st);
// ---- stage-pipelined CG SpMV (ep_staged.cu): structured 27-point graph, symmetric storage
constexpr int kStageMaxUpper = 14;   // stored slots per row (diagonal + 13 upper)
constexpr int kStageMaxRow = 27;     // entries per row
constexpr int kStageMaxGlobal = 13;  // leading entries that may live in an earlier stage

struct StageDesc {
  int R0, R1;        // rows [R0, R1) of the stage
  int slot0, slot1;  // stored slots of those rows (symmetric storage)
  int64_t blk_off;   // index block (bytes, 16-aligned)
  int blk_bytes;
  int g;             // canonical stage id (tiles g*T ...); desc is stored in sweep order
};

struct StageMap {
  int nstages = 0, s = 0, N = 0;
  int xlo = 0, xhi = 0;  // rows of p the x runs may read: [xlo, xhi) (slab: ghost planes included)
  TileMap tm{};
  StageDesc* desc = nullptr;
  unsigned char* blk = nullptr;
  int64_t blk_bytes = 0;
  int idx_bytes = 0;   // one stage's index block
  int n_interior = 0;  // slabs: the first n_interior sweep positions read no ghost plane
};

bool staged_supported(int s, int N);
// N = mesh nodes per axis (rows == N^3, the k_build_graph numbering); up_start =
// first stored slot of each row (rows + 1). Fails (InvalidValue) for graphs
// that are not the structured 27-point pattern.
// Slabs: tm.rows is a multiple of N^2 (owned planes), columns and the x runs
// may reach [xlo, xhi) (defaults: [0, tm.rows)).
cudaError_t build_stage_map(int s, const TileMap& tm, int N, const int* row_map,
                            const int* col_entry, const int* vpos, const int* up_start,
                            StageMap& sm, cudaStream_t st, int xlo = 0, int xhi = -1,
                            int interior_lo = 0, int interior_hi = -1);
void free_stage_map(StageMap& sm);
// Halo overlap (slabs): with interior_lo < interior_hi, the stages whose rows
// all lie in [interior_lo, interior_hi) go first in the sweep (n_interior of
// them). Their x runs then stay inside the owned rows, so they can run while
// the ghost planes are in flight. stage_range views sweep positions
// [pos0, pos0 + count) as a map of its own, with x runs clipped to [xlo, xhi).
StageMap stage_range(const StageMap& sm, int pos0, int count, int xlo, int xhi);
// q = A p and (tiles) the canonical p.q tile partials; bitwise equal to the
// warp-per-tile kernel
// fuse_fin (tiles only): the kernel also runs the canonical finalize of p.q
// (k_fin_segments' work and order) after a grid barrier (f.bar), so no
// separate finalize launch follows. Stages are claimed dynamically through
// f.ticket (zero between launches). Without tiles, f.prod (if set) receives
// the per-row products p*q for the serial-order chain.
cudaError_t launch_cg_spmv_staged(int s, bool tiles, bool fuse_fin, const StageMap& sm,
                                  const double* values, const double* p, double* q, const FinArgs& f,
                                  cudaStream_t st);
bool staged_fuse_fin();  // ENPROP_STAGED_FUSE (env, default 1)
bool staged_serial();    // ENPROP_STAGED_SERIAL (env, default 1)
bool plain_cg_spmv();    // ENPROP_PLAIN_CG_SPMV (env, default 1): public SpMV kernels in unstaged full-storage CG
int spmv_variant();  // ENPROP_OPT_SPMV_VARIANT of the calling context (-1 = auto)

// after the loop: apply the still-deferred x += alpha*p of the last iteration
cudaError_t launch_cg_flush(int s, int rows, double* x, double* const* p, const CgState* cg,
                            cudaStream_t st);

}  // namespace ep
