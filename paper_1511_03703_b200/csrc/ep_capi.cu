// C ABI of enprop_b200 (include/enprop_b200.h). Host orchestration only: all
// arithmetic on the hot path runs in the sm_100a kernels of ep_kernels.cu /
// ep_assemble.cu. There is no CPU fallback: a missing or failing device is an
// ENPROP_ERR_CUDA.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "enprop_b200.h"
#include "ep_host.h"
#include "ep_internal.h"
#include "ep_kernels.h"

using namespace ep;
using namespace ep_internal;

namespace ep_internal {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t err, const char* where) {
  return fail(err == cudaErrorMemoryAllocation ? ENPROP_ERR_OOM : ENPROP_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(err));
}

bool valid_width(int s) { return s == 1 || s == 2 || s == 4 || s == 8 || s == 16 || s == 32; }
}  // namespace ep_internal

namespace {

// Workspace of one CG solve on `rows` x s.
struct CgWork {
  double* r = nullptr;
  double* p[2] = {nullptr, nullptr};
  double* q = nullptr;
  double* partials = nullptr;  // canonical tile partials [tiles][s]
  double* seg_sums = nullptr;  // [segs][s]
  int* counters = nullptr;     // kCounterInts counter words (ep_kernels.h)
  double* prod = nullptr;      // serial order: p*q products [rows][s] (allocated on first use)
  double* hist = nullptr;
  CgState* state = nullptr;
  int rows = 0, s = 0, maxit = -1, tiles = 0, segs = 0;
  // CUDA graph of one chunk of CG iterations (ENPROP_OPT_GRAPHS), replayed for
  // every full chunk that starts at an even iteration; rebuilt when any
  // pointer or schedule choice baked into its launches changes
  cudaGraphExec_t graph = nullptr;
  std::vector<char> graph_key;
};

void free_graph(CgWork& w) {
  if (w.graph) cudaGraphExecDestroy(w.graph);
  w.graph = nullptr;
  w.graph_key.clear();
}

void free_work(CgWork& w) {
  free_graph(w);
  for (void* p : {(void*)w.r, (void*)w.p[0], (void*)w.p[1], (void*)w.q, (void*)w.partials,
                  (void*)w.seg_sums, (void*)w.counters, (void*)w.prod, (void*)w.hist,
                  (void*)w.state})
    if (p) cudaFree(p);
  w = CgWork{};
}

int ensure_work(CgWork& w, int rows, int s, int maxit, const TileMap& tm, bool need_prod) {
  const int tiles = tm.num_tiles() > 0 ? tm.num_tiles() : 1;
  const int segs = tm.num_segs > 0 ? tm.num_segs : 1;
  const size_t vec = (size_t)rows * s * sizeof(double);
  const size_t vb = vec > 0 ? vec : 8;
  if (w.r && w.rows == rows && w.s == s && w.maxit >= maxit && w.tiles >= tiles && w.segs >= segs) {
    if (need_prod && !w.prod) EP_CUDA(cudaMalloc(&w.prod, vb));
    return ENPROP_OK;
  }
  free_work(w);
  if (need_prod) EP_CUDA(cudaMalloc(&w.prod, vb));
  EP_CUDA(cudaMalloc(&w.r, vb));
  EP_CUDA(cudaMalloc(&w.p[0], vb));
  EP_CUDA(cudaMalloc(&w.p[1], vb));
  EP_CUDA(cudaMalloc(&w.q, vb));
  EP_CUDA(cudaMalloc(&w.partials, (size_t)tiles * s * sizeof(double)));
  EP_CUDA(cudaMalloc(&w.seg_sums, (size_t)segs * s * sizeof(double)));
  EP_CUDA(cudaMalloc(&w.counters, kCounterInts * sizeof(int)));
  EP_CUDA(cudaMemset(w.counters, 0, kCounterInts * sizeof(int)));
  EP_CUDA(cudaMalloc(&w.hist, (size_t)(maxit + 1) * s * sizeof(double)));
  EP_CUDA(cudaMalloc(&w.state, sizeof(CgState)));
  w.rows = rows;
  w.s = s;
  w.maxit = maxit;
  w.tiles = tiles;
  w.segs = segs;
  return ENPROP_OK;
}

FinArgs fin_args(const CgWork& w, int phase) {
  FinArgs f;
  f.partials = w.partials;
  f.seg_sums = w.seg_sums;
  f.seg_done = w.counters;
  f.bar = w.counters + 1;
  f.ticket = w.counters + 3;
  f.prod = w.prod;
  f.phase = phase;
  f.cg = w.state;
  f.hist = w.hist;
  f.lanes_out = nullptr;
  f.seg_only = 0;
  f.defer = 1;
  return f;
}

int validate_cg_options(const enprop_cg_options* opt, int s) {
  if (!opt) return fail(ENPROP_ERR_INVALID, "enprop_cg: options are required");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (opt->flavour != ENPROP_CG_COUPLED && opt->flavour != ENPROP_CG_UNCOUPLED)
    return fail(ENPROP_ERR_INVALID, "enprop_cg: unknown CG flavour");
  if (opt->dot_mode != ENPROP_DOT_SERIAL && opt->dot_mode != ENPROP_DOT_CANONICAL)
    return fail(ENPROP_ERR_INVALID, "enprop_cg: unknown dot mode");
  if (opt->max_iterations < 0) return fail(ENPROP_ERR_INVALID, "enprop_cg: negative max_iterations");
  return ENPROP_OK;
}

// Six events per profiled iteration (grown on demand, reused across solves):
// before the direction pass, before the SpMV, after it, after the PQ finalize,
// after the update, after the RR finalize.
constexpr int kProfEv = 6;
cudaEvent_t* prof_slot(enprop_ctx* c) {
  if (c->prof_used + kProfEv > c->prof_ev.size()) {
    for (int k = 0; k < 32 * kProfEv; ++k) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      c->prof_ev.push_back(e);
    }
  }
  cudaEvent_t* p = &c->prof_ev[c->prof_used];
  c->prof_used += kProfEv;
  return p;
}

// Accumulate the recorded iterations: the first `working` did work; the rest
// were enqueued past convergence and early-exited (their time goes to [8]).
int prof_collect(enprop_ctx* c, int working) {
  for (size_t i = 0; i + kProfEv <= c->prof_used; i += kProfEv) {
    float t[kProfEv - 1];
    for (int k = 0; k + 1 < kProfEv; ++k)
      EP_CUDA(cudaEventElapsedTime(&t[k], c->prof_ev[i + k], c->prof_ev[i + k + 1]));
    const float all = t[0] + t[1] + t[2] + t[3] + t[4];
    if ((int)(i / kProfEv) < working) {
      c->prof_ms += t[1];
      c->prof_count += 1;
      c->prof_detail[0] += t[0] + t[1];
      c->prof_detail[1] += t[2];
      c->prof_detail[2] += t[3];
      c->prof_detail[3] += t[4];
      c->prof_detail[4] += all;
      c->prof_detail[9] += t[0];
      c->prof_detail[10] += t[1];
    } else {
      c->prof_detail[8] += all;
    }
  }
  c->prof_used = 0;
  return ENPROP_OK;
}

// The CG driver (pcg.hpp:52-103 semantics; see ep_kernels.cu cg_phase).
// Iterations are enqueued in chunks of check_every; the host reads the
// device's `done` flag of chunk c while chunk c+1 is already queued, so the GPU
// never idles on the check. Kernels of iterations past convergence early-exit.
int run_cg(enprop_ctx* ctx, int s, int rows, const int* row_map, const int* col_entry,
           const double* values, const double* b, double* x, const enprop_cg_options* opt,
           CgWork& w, int* iterations, int* lane_status, double* history, int* hist_len,
           const int* vpos = nullptr, const StageMap* stage = nullptr) {
  const int seg = opt->seg_rows > 0 ? opt->seg_rows : 4096;
  const TileMap tm = make_tile_map(rows, seg);
  const bool canon = opt->dot_mode == ENPROP_DOT_CANONICAL;
  // serial order: the SpMV writes the p*q products the chain kernel sums
  // (except on the plain path, where the chain forms them from p and q; a
  // chain reading p and q everywhere measured 0.5-0.7% slower at 24 groups)
  int rc = ensure_work(w, rows, s, opt->max_iterations, tm, !canon);
  if (rc) return rc;
  const int lanes = opt->flavour == ENPROP_CG_UNCOUPLED ? s : 1;
  const bool fused = ctx->fused_direction != 0 && vpos == nullptr;  // symmetric storage: split only
  cudaStream_t st = ctx->stream;
  cudaEvent_t* sev = nullptr;  // profiled: solve start, loop start, loop end, solve end
  if (ctx->profile) {
    if (!ctx->prof_solve_ev[0])
      for (int k = 0; k < 4; ++k) EP_CUDA(cudaEventCreate(&ctx->prof_solve_ev[k]));
    sev = ctx->prof_solve_ev;
    EP_CUDA(cudaEventRecord(sev[0], st));
  }

  CgState init;
  std::memset(&init, 0, sizeof(init));
  init.flavour = opt->flavour;
  init.s = s;
  init.maxit = opt->max_iterations;
  init.tol = opt->tol;
  EP_CUDA(cudaMemcpyAsync(w.state, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  const size_t vec = (size_t)rows * s * sizeof(double);
  if (vec) {
    EP_CUDA(cudaMemsetAsync(x, 0, vec, st));
    EP_CUDA(cudaMemcpyAsync(w.r, b, vec, cudaMemcpyDeviceToDevice, st));
  }
  const FinArgs f_init = fin_args(w, kPhaseInit);
  const FinArgs f_pq = fin_args(w, kPhasePQ);
  const FinArgs f_rr = fin_args(w, kPhaseRR);
  const bool fin_kernel = canon;
  // the staged SpMV finalizes p.q itself (grid barrier)
  const bool fuse_pq = stage && canon && staged_fuse_fin() && tm.num_segs >= 1;
  if (canon) {
    EP_CUDA(launch_dot_tiles(s, tm, w.r, w.r, f_init, st));
    if (fin_kernel) EP_CUDA(launch_fin_segments(s, tm, f_init, st));
    ctx->launches += fin_kernel ? 2 : 1;
  } else {  // b_norm = norm2(b), rz = dot(r, z) (pcg.hpp:62-73): one chain over r = b
    EP_CUDA(launch_chain(s, rows, w.r, nullptr, kChainSquare, f_init, st));
    ctx->launches += 1;
  }

  if (sev) EP_CUDA(cudaEventRecord(sev[1], st));
  const int chunk = opt->check_every > 0 ? opt->check_every : 16;
  // Full storage without the staged kernel: q = A p by the public SpMV kernels
  // (k_spmv_small for s <= 16: one CTA stages its block's column indices;
  // k_spmv at s = 32), then p.q as its own pass -- canonical tile partials
  // (k_dot_tiles) or the serial chain over p and q. The warp-per-tile CG
  // kernel (SpMV + tile trees in one pass) stays for symmetric storage and the
  // fused-direction schedule. (64^3, s = 1: 0.077 -> ~0.03 ms per SpMV.)
  const bool plain = !stage && !vpos && !fused && plain_cg_spmv();
  const int per_iter = (canon ? 2 : 4) + (fused ? 0 : 1) + (fin_kernel ? 2 : 0) - (fuse_pq ? 1 : 0) +
                       (plain && canon ? 1 : 0);
  // one loop body (pcg.hpp:76-101); `it` fixes which p buffer is old / new
  auto enqueue_iteration = [&](int it, cudaEvent_t* ev) -> cudaError_t {
    double* p_old = w.p[it & 1];
    double* p_new = w.p[(it + 1) & 1];
    cudaError_t e = cudaSuccess;
#define EP_Q(call)                 \
  do {                             \
    if ((e = (call)) != cudaSuccess) \
      return e;                    \
  } while (0)
    if (ev) EP_Q(cudaEventRecord(ev[0], st));
    if (!fused) EP_Q(launch_cg_direction(s, rows, w.r, p_old, p_new, x, w.state, st));
    if (ev) EP_Q(cudaEventRecord(ev[1], st));
    if (stage) {
      EP_Q(launch_cg_spmv_staged(s, canon, fuse_pq, *stage, values, p_new, w.q, f_pq, st));
    } else if (plain) {
      if (s <= spmv_small_max())
        EP_Q(launch_spmv_small(s, rows, row_map, col_entry, values, p_new, w.q, st));
      else
        EP_Q(launch_spmv(s, rows, row_map, col_entry, values, p_new, w.q, false, st));
      if (canon) EP_Q(launch_dot_tiles(s, tm, p_new, w.q, f_pq, st));
    } else {
      EP_Q(launch_cg_spmv(s, canon, fused, false, tm, row_map, col_entry, values, w.r, p_old, p_new, w.q,
                          x, p_new, vpos, f_pq, st));
    }
    if (ev) EP_Q(cudaEventRecord(ev[2], st));
    if (!canon) {
      if (plain || !w.prod) EP_Q(launch_chain(s, rows, p_new, w.q, kChainProduct, f_pq, st));
      else EP_Q(launch_chain(s, rows, w.prod, nullptr, kChainGiven, f_pq, st));
    }
    if (fin_kernel && !fuse_pq) EP_Q(launch_fin_segments(s, tm, f_pq, st));
    if (ev) EP_Q(cudaEventRecord(ev[3], st));
    EP_Q(launch_cg_update(s, canon, tm, w.r, w.q, f_rr, st));
    if (ev) EP_Q(cudaEventRecord(ev[4], st));
    if (!canon) EP_Q(launch_chain(s, rows, w.r, nullptr, kChainSquare, f_rr, st));
    if (fin_kernel) EP_Q(launch_fin_segments(s, tm, f_rr, st));
    if (ev) EP_Q(cudaEventRecord(ev[5], st));
#undef EP_Q
    return cudaSuccess;
  };
  // CUDA graph of a whole chunk (ENPROP_OPT_GRAPHS): one launch per chunk
  // instead of per_iter * chunk; captured on this thread only, after the
  // first chunk ran eagerly (which performed any one-time kernel attribute
  // setup). Everything a replay depends on is part of the key.
  bool use_graph = ctx->graphs && !ctx->profile && chunk % 2 == 0;
  if (use_graph) {
    const void* key_ptrs[] = {values, x, row_map, col_entry, vpos, stage ? (const void*)stage->desc : nullptr,
                              w.r, w.q, w.p[0], w.p[1], w.prod, w.partials, w.state};
    const int key_ints[] = {s, rows, canon, fuse_pq, fused, chunk, tm.seg_rows, launch_opts().pdl,
                            spmv_variant(), plain};
    std::vector<char> key(sizeof(key_ptrs) + sizeof(key_ints));
    std::memcpy(key.data(), key_ptrs, sizeof(key_ptrs));
    std::memcpy(key.data() + sizeof(key_ptrs), key_ints, sizeof(key_ints));
    if (w.graph && w.graph_key != key) free_graph(w);
    w.graph_key = key;
  }
  auto capture_chunk = [&]() -> bool {  // false: run eagerly instead
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaError_t e = cudaSuccess;
    for (int c = 0; c < chunk && e == cudaSuccess; ++c) e = enqueue_iteration(c, nullptr);
    const cudaError_t e2 = cudaStreamEndCapture(st, &g);
    if (e == cudaSuccess && e2 == cudaSuccess && g &&
        cudaGraphInstantiate(&w.graph, g, 0) == cudaSuccess) {
      cudaGraphDestroy(g);
      return true;
    }
    if (g) cudaGraphDestroy(g);
    w.graph = nullptr;
    cudaGetLastError();  // capture unsupported here: eager launches
    return false;
  };
  int launched = 0;
  int slot = 0;
  bool pending = false;
  const int limit = opt->max_iterations;  // loop bodies that can run (pcg.hpp:79-85)
  while (true) {
    if (launched < limit) {
      if (use_graph && launched > 0 && launched % 2 == 0 && launched + chunk <= limit &&
          (w.graph || capture_chunk())) {
        EP_CUDA(cudaGraphLaunch(w.graph, st));
        launched += chunk;
        ctx->launches += (int64_t)per_iter * chunk;
      } else {
        if (use_graph && !w.graph && launched > 0) use_graph = false;  // capture failed
        for (int c = 0; c < chunk && launched < limit; ++c, ++launched) {
          cudaEvent_t* ev = ctx->profile ? prof_slot(ctx) : nullptr;
          EP_CUDA(enqueue_iteration(launched, ev));
          ctx->launches += per_iter;
        }
      }
    }
    // flag of this chunk
    EP_CUDA(cudaMemcpyAsync(&ctx->pinned_flags[slot], &w.state->done, sizeof(int),
                            cudaMemcpyDeviceToHost, st));
    EP_CUDA(cudaEventRecord(ctx->flag_ev[slot], st));
    if (pending) {  // previous chunk's flag
      EP_CUDA(cudaEventSynchronize(ctx->flag_ev[slot ^ 1]));
      if (ctx->pinned_flags[slot ^ 1]) break;
    }
    if (launched >= limit) {
      EP_CUDA(cudaEventSynchronize(ctx->flag_ev[slot]));
      break;
    }
    pending = true;
    slot ^= 1;
  }
  if (sev) EP_CUDA(cudaEventRecord(sev[2], st));
  // the last finished iteration's x += alpha*p is still deferred
  EP_CUDA(launch_cg_flush(s, rows, x, w.p, w.state, st));
  ctx->launches += 1;
  if (sev) EP_CUDA(cudaEventRecord(sev[3], st));
  EP_CUDA(cudaStreamSynchronize(st));

  CgState fin;
  EP_CUDA(cudaMemcpy(&fin, w.state, sizeof(fin), cudaMemcpyDeviceToHost));
  if (ctx->profile) {
    rc = prof_collect(ctx, fin.it);
    if (rc) return rc;
    float t[3];
    EP_CUDA(cudaEventElapsedTime(&t[0], sev[0], sev[3]));
    EP_CUDA(cudaEventElapsedTime(&t[1], sev[0], sev[1]));
    EP_CUDA(cudaEventElapsedTime(&t[2], sev[1], sev[2]));
    for (int k = 0; k < 3; ++k) ctx->prof_detail[5 + k] += t[k];
  }
  if (!fin.done) return fail(ENPROP_ERR_CUDA, "enprop_cg: solver did not finish (internal)");
  for (int l = 0; l < lanes; ++l) {
    if (iterations) iterations[l] = fin.iters[l];
    if (lane_status) lane_status[l] = opt->flavour == ENPROP_CG_UNCOUPLED ? fin.lane_status[l] : fin.status;
    if (hist_len) hist_len[l] = fin.hist_len[l];
  }
  if (history) {  // copy only the recorded rows; NaN past each lane's end
    int len = 0;
    for (int l = 0; l < lanes; ++l) len = fin.hist_len[l] > len ? fin.hist_len[l] : len;
    std::vector<double> h((size_t)len * lanes);
    if (len) EP_CUDA(cudaMemcpy(h.data(), w.hist, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int it = 0; it <= opt->max_iterations; ++it)
      for (int l = 0; l < lanes; ++l)
        history[(size_t)it * lanes + l] = it < fin.hist_len[l] ? h[(size_t)it * lanes + l] : NAN;
  }

  if (fin.status == ENPROP_ERR_NO_CONVERGENCE)
    return fail(ENPROP_ERR_NO_CONVERGENCE, "pcg_solve: no convergence within " +
                                               std::to_string(opt->max_iterations) + " iterations");
  if (fin.status == ENPROP_ERR_INDEFINITE)
    return fail(ENPROP_ERR_INDEFINITE, "pcg_solve: operator not positive definite (p'Ap <= 0)");
  return ENPROP_OK;
}

}  // namespace

// ============================================================================
extern "C" {

const char* enprop_last_error(void) { return g_last_error.c_str(); }
int enprop_abi_version(void) { return ENPROP_ABI_VERSION; }

int enprop_ctx_create(int device, enprop_ctx** out) {
  if (!out) return fail(ENPROP_ERR_INVALID, "enprop_ctx_create: null output");
  int count = 0;
  cudaError_t err = cudaGetDeviceCount(&count);
  if (err != cudaSuccess || count == 0)
    return fail(ENPROP_ERR_CUDA, "enprop_ctx_create: no CUDA device (enprop_b200 has no CPU path)");
  if (device < 0 || device >= count) return fail(ENPROP_ERR_INVALID, "enprop_ctx_create: bad device");
  EP_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  EP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(ENPROP_ERR_CUDA, "enprop_ctx_create: enprop_b200 is built for sm_100a (B200) only");
  auto* c = new (std::nothrow) enprop_ctx();
  if (!c) return fail(ENPROP_ERR_OOM, "enprop_ctx_create: out of host memory");
  c->device = device;
  // ENPROP_GRAPHS=0 (env) makes "off" the default of ENPROP_OPT_GRAPHS: Nsight
  // Compute 2025.2.1 aborts with host heap corruption when many threads capture and
  // replay CUDA graphs concurrently (24-group bench, graphs on; clean with them
  // off, and clean without the profiler under MALLOC_CHECK_=3), so profiling
  // runs launch kernel by kernel
  c->graphs = env_int("ENPROP_GRAPHS", 1) != 0 ? 1 : 0;
  EP_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  EP_CUDA(cudaMallocHost(&c->pinned_flags, 2 * sizeof(int)));
  EP_CUDA(cudaEventCreateWithFlags(&c->flag_ev[0], cudaEventDisableTiming));
  EP_CUDA(cudaEventCreateWithFlags(&c->flag_ev[1], cudaEventDisableTiming));
  *out = c;
  return ENPROP_OK;
}

int enprop_ctx_destroy(enprop_ctx* c) {
  if (!c) return ENPROP_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->flag_ev[0]) cudaEventDestroy(c->flag_ev[0]);
  if (c->flag_ev[1]) cudaEventDestroy(c->flag_ev[1]);
  if (c->pinned_flags) cudaFreeHost(c->pinned_flags);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof_solve_ev)
    if (e) cudaEventDestroy(e);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return ENPROP_OK;
}

int enprop_ctx_set_stream(enprop_ctx* c, void* stream) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  c->stream = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
  return ENPROP_OK;
}

void* enprop_ctx_stream(enprop_ctx* c) { return c ? (void*)c->stream : nullptr; }

int enprop_ctx_synchronize(enprop_ctx* c) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  EP_CUDA(cudaStreamSynchronize(c->stream));
  return ENPROP_OK;
}

int64_t enprop_ctx_launch_count(enprop_ctx* c) { return c ? c->launches : 0; }

int enprop_ctx_set_option(enprop_ctx* c, int option, int value) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  switch (option) {
    case ENPROP_OPT_FUSED_DIRECTION:
      c->fused_direction = value ? 1 : 0;
      return ENPROP_OK;
    case ENPROP_OPT_SPMV_PIPELINE:
      c->spmv_pipeline = value ? 1 : 0;
      return ENPROP_OK;
    case ENPROP_OPT_SYMMETRIC_STORAGE:
      c->symmetric_storage = value < 0 ? 0 : (value > 2 ? 2 : value);
      return ENPROP_OK;
    case ENPROP_OPT_SPMV_VARIANT:
      c->spmv_variant = (value >= 0 && value <= 6) ? value : -1;
      return ENPROP_OK;
    case ENPROP_OPT_PDL:
      c->pdl = value ? 1 : 0;
      return ENPROP_OK;
    case ENPROP_OPT_GRAPHS:
      c->graphs = value ? 1 : 0;
      return ENPROP_OK;

    default:
      return fail(ENPROP_ERR_INVALID, "enprop_ctx_set_option: unknown option");
  }
}

int enprop_ctx_profile(enprop_ctx* c, int enable, double* spmv_ms, int64_t* spmv_launches) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (spmv_ms) *spmv_ms = c->prof_ms;
  if (spmv_launches) *spmv_launches = c->prof_count;
  if (enable >= 0) {
    c->profile = enable;
    c->prof_ms = 0.0;
    c->prof_count = 0;
    for (double& d : c->prof_detail) d = 0.0;
  }
  return ENPROP_OK;
}

int enprop_ctx_profile_detail(enprop_ctx* c, double* ms, int64_t* iterations) {
  if (!c || !ms) return fail(ENPROP_ERR_INVALID, "enprop_ctx_profile_detail: null argument");
  for (int k = 0; k < 11; ++k) ms[k] = c->prof_detail[k];
  if (iterations) *iterations = c->prof_count;
  return ENPROP_OK;
}

int enprop_malloc(enprop_ctx* c, size_t bytes, void** dptr) {
  if (!c || !dptr) return fail(ENPROP_ERR_INVALID, "enprop_malloc: null argument");
  EP_CUDA(cudaSetDevice(c->device));
  EP_CUDA(cudaMalloc(dptr, bytes ? bytes : 8));
  return ENPROP_OK;
}

int enprop_free(enprop_ctx* c, void* dptr) {
  if (!c) return fail(ENPROP_ERR_INVALID, "enprop_free: null context");
  if (dptr) EP_CUDA(cudaFree(dptr));
  return ENPROP_OK;
}

int enprop_memcpy_h2d(enprop_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (!bytes) return ENPROP_OK;
  EP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  EP_CUDA(cudaStreamSynchronize(c->stream));
  return ENPROP_OK;
}

int enprop_memcpy_d2h(enprop_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (!bytes) return ENPROP_OK;
  EP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  EP_CUDA(cudaStreamSynchronize(c->stream));
  return ENPROP_OK;
}

int64_t enprop_mesh_nnz(int n) {
  if (n < 1) return 0;
  const int64_t t = 3 * (int64_t)(n + 1) - 2;
  return t * t * t;
}

int enprop_build_node_graph(enprop_ctx* c, int n, int* row_map, int* col_entry) {
  if (!c || !row_map || !col_entry) return fail(ENPROP_ERR_INVALID, "enprop_build_node_graph: null argument");
  if (n < 1) return fail(ENPROP_ERR_INVALID, "StructuredMesh: cells_per_axis must be at least 1");
  if (enprop_mesh_nnz(n) > 2147483647LL)
    return fail(ENPROP_ERR_INVALID, "enprop_build_node_graph: nnz exceeds int32 (reference Graph uses int)");
  EP_CUDA(launch_build_graph(n, row_map, col_entry, c->stream));
  c->launches += 1;
  return ENPROP_OK;
}

int enprop_draw_samples(uint64_t seed, int count, int m, double* out) {
  if (m < 1) return fail(ENPROP_ERR_INVALID, "draw_samples: need at least one coordinate");
  if (count < 0) return fail(ENPROP_ERR_INVALID, "draw_samples: negative count");
  if (count > 0 && !out) return fail(ENPROP_ERR_INVALID, "draw_samples: null output");
  std::mt19937_64 rng(seed);  // samples.cpp:11-16: top 53 bits -> [0,1) -> [-1,1)
  for (int64_t i = 0; i < (int64_t)count * m; ++i)
    out[i] = double(rng() >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  return ENPROP_OK;
}

int enprop_pack_sample_group(const double* samples, int count, int m, int group_start, int s,
                             double* out) {
  if (group_start < 0 || s < 1 || group_start + s > count)
    return fail(ENPROP_ERR_INVALID, "pack_sample_group: not enough samples for the group");
  if (m < 1 || !samples || !out) return fail(ENPROP_ERR_INVALID, "pack_sample_group: bad argument");
  for (int j = 0; j < m; ++j)
    for (int e = 0; e < s; ++e) out[(size_t)j * s + e] = samples[(size_t)(group_start + e) * m + j];
  return ENPROP_OK;
}

int enprop_kl_describe(const enprop_kl_params* kl, int* mode_axes, double* mode_eigenvalue,
                       double* axis_frequency, double* axis_eigenvalue, double* axis_inverse_norm,
                       int* axis_cosine) {
  if (!kl) return fail(ENPROP_ERR_INVALID, "enprop_kl_describe: null params");
  KlHost f;
  if (!kl_init(f, kl->num_terms, kl->mean, kl->sigma, kl->correlation_length))
    return fail(ENPROP_ERR_INVALID, "KlField: invalid num_terms/mean/sigma/correlation_length");
  for (int i = 0; i < f.m; ++i) {
    if (mode_axes)
      for (int a = 0; a < 3; ++a) mode_axes[i * 3 + a] = f.mode_axes[i * 3 + a];
    if (mode_eigenvalue) mode_eigenvalue[i] = f.mode_eig[i];
    if (axis_frequency) axis_frequency[i] = f.axis_freq[i];
    if (axis_eigenvalue) axis_eigenvalue[i] = f.axis_eig[i];
    if (axis_inverse_norm) axis_inverse_norm[i] = f.axis_invnorm[i];
    if (axis_cosine) axis_cosine[i] = f.axis_cos[i];
  }
  return ENPROP_OK;
}

}  // extern "C"

namespace ep_internal {


int make_asm_setup(enprop_ctx* c, int n, const enprop_kl_params* kl,
                   const enprop_pde_coeffs* coeffs, AsmSetup& out) {
  if (n < 1) return fail(ENPROP_ERR_INVALID, "StructuredMesh: cells_per_axis must be at least 1");
  KlHost f;
  if (!kl || !kl_init(f, kl->num_terms, kl->mean, kl->sigma, kl->correlation_length))
    return fail(ENPROP_ERR_INVALID, "KlField: invalid num_terms/mean/sigma/correlation_length");
  const std::vector<double> F = kl_axis_tables(f, n);
  AsmTables T;
  const double zero_v[3] = {1.0, 0.0, 0.0};
  make_asm_tables(T, n, coeffs ? coeffs->alpha : 0.0, coeffs ? coeffs->beta : 0.0,
                  coeffs ? coeffs->velocity : zero_v);
  EP_CUDA(cudaMalloc(&out.F, F.size() * sizeof(double)));
  EP_CUDA(cudaMalloc(&out.tab, sizeof(AsmTables)));
  EP_CUDA(cudaMemcpyAsync(out.F, F.data(), F.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  EP_CUDA(cudaMemcpyAsync(out.tab, &T, sizeof(T), cudaMemcpyHostToDevice, c->stream));
  EP_CUDA(cudaStreamSynchronize(c->stream));  // host sources go out of scope
  AsmArgs& a = out.args;
  std::memset(&a, 0, sizeof(a));
  a.n = n;
  a.rows = (n + 1) * (n + 1) * (n + 1);
  a.m = f.m;
  a.mean = f.mean;
  a.F = out.F;
  a.tab = out.tab;
  a.T = T;
  a.nonlinear = (coeffs && (coeffs->alpha != 0.0 || coeffs->beta != 0.0)) ? 1 : 0;
  for (int i = 0; i < f.m; ++i) {
    for (int k = 0; k < 3; ++k) a.mode_axes[i][k] = f.mode_axes[i * 3 + k];
    a.mode_sl[i] = f.sigma * f.mode_sqrt_eig[i];  // kl.hpp:74: sigma * sqrt_eigenvalue first
  }
  return ENPROP_OK;
}

void free_asm_setup(AsmSetup& s) {
  if (s.F) cudaFree(s.F);
  if (s.tab) cudaFree(s.tab);
  s = AsmSetup{};
}

}  // namespace ep_internal

extern "C" {

int enprop_assemble(enprop_ctx* c, int s, int n, const enprop_kl_params* kl,
                    const enprop_pde_coeffs* coeffs, const double* u, const double* y,
                    const int* row_map, double* values, double* residual,
                    const enprop_dirichlet_bc* bc) {
  if (!c || !y || !row_map || !values || !residual)
    return fail(ENPROP_ERR_INVALID, "enprop_assemble: null argument");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  AsmSetup setup;
  int rc = make_asm_setup(c, n, kl, coeffs, setup);
  if (rc) {
    free_asm_setup(setup);
    return rc;
  }
  AsmArgs a = setup.args;
  a.u = u;
  a.y = y;
  a.row_map = row_map;
  a.values = values;
  a.residual = residual;
  a.dirichlet = bc ? 1 : 0;
  a.bc0 = bc ? bc->x0_value : 1.0;
  a.bc1 = bc ? bc->x1_value : 0.0;
  cudaError_t err = launch_assemble(s, a, c->stream);
  c->launches += 1;
  if (err == cudaSuccess) err = cudaStreamSynchronize(c->stream);  // tables are freed below
  free_asm_setup(setup);
  if (err != cudaSuccess) return cuda_fail(err, "enprop_assemble");
  return ENPROP_OK;
}

int enprop_apply_dirichlet(enprop_ctx* c, int s, int n, const enprop_dirichlet_bc* bc,
                           const int* row_map, const int* col_entry, const double* u,
                           double* values, double* residual) {
  if (!c || !bc || !row_map || !col_entry || !values || !residual)
    return fail(ENPROP_ERR_INVALID, "enprop_apply_dirichlet: null argument");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (n < 1) return fail(ENPROP_ERR_INVALID, "StructuredMesh: cells_per_axis must be at least 1");
  EP_CUDA(launch_dirichlet(s, n, bc->x0_value, bc->x1_value, row_map, col_entry, u, values, residual,
                           c->stream));
  c->launches += 1;
  return ENPROP_OK;
}

int enprop_spmv(enprop_ctx* c, int s, int rows, int cols, const int* row_map,
                const int* col_entry, const double* values, const double* x, double* z) {
  ScopedLaunchOpts launch_scope(c);
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (rows < 0 || cols < 0) return fail(ENPROP_ERR_INVALID, "spmv: negative dimension");
  if (rows == 0) return ENPROP_OK;
  if (!row_map || !z || (cols > 0 && !x)) return fail(ENPROP_ERR_INVALID, "spmv: null argument");
  if (s <= spmv_small_max() && !c->spmv_pipeline)  // narrow rows: shared-memory staged blocks (ep_outer.cu)
    EP_CUDA(launch_spmv_small(s, rows, row_map, col_entry, values, x, z, c->stream));
  else
    EP_CUDA(launch_spmv(s, rows, row_map, col_entry, values, x, z, c->spmv_pipeline != 0, c->stream));
  c->launches += 1;
  return ENPROP_OK;
}

int enprop_spmv_small_config(int s, int* routed, int* threads, int* reg_cap, int* stage_mode) {
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (routed) *routed = s <= spmv_small_max();
  spmv_small_config(s, threads, reg_cap, stage_mode);
  return ENPROP_OK;
}

int enprop_spmv_outer(enprop_ctx* c, int s, int rows, int cols, int64_t nnz, const int* row_map,
                      const int* col_entry, const double* values, const double* x, double* z) {
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (s < 1) return fail(ENPROP_ERR_INVALID, "spmv_outer: ensemble_size must be at least 1");
  if (rows < 0 || cols < 0 || nnz < 0) return fail(ENPROP_ERR_INVALID, "spmv_outer: negative dimension");
  if (rows == 0) return ENPROP_OK;
  if (!row_map || !z || (cols > 0 && !x) || (nnz > 0 && (!col_entry || !values)))
    return fail(ENPROP_ERR_INVALID, "spmv_outer: null argument");
  EP_CUDA(launch_spmv_outer(s, rows, cols, nnz, row_map, col_entry, values, x, z, c->stream));
  c->launches += 1;
  return ENPROP_OK;
}

int enprop_dot(enprop_ctx* c, int s, int64_t n, const double* u, const double* v, int dot_mode,
               int seg_rows, double* lanes_host, double* coupled_host) {
  ScopedLaunchOpts launch_scope(c);
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (n < 0 || n > 2147483647LL) return fail(ENPROP_ERR_INVALID, "dot: bad length");
  double* out = nullptr;
  const int rows = (int)n;
  const TileMap tm = make_tile_map(rows, seg_rows > 0 ? seg_rows : 4096);
  CgWork w;  // partials + counters only
  cudaError_t err = cudaMalloc(&out, (s + 1) * sizeof(double));
  const int tiles = tm.num_tiles() > 0 ? tm.num_tiles() : 1;
  const int segs = tm.num_segs > 0 ? tm.num_segs : 1;
  if (err == cudaSuccess) err = cudaMalloc(&w.partials, (size_t)tiles * s * sizeof(double));
  if (err == cudaSuccess) err = cudaMalloc(&w.seg_sums, (size_t)segs * s * sizeof(double));
  if (err == cudaSuccess) err = cudaMalloc(&w.counters, kCounterInts * sizeof(int));
  if (err == cudaSuccess) err = cudaMemsetAsync(w.counters, 0, kCounterInts * sizeof(int), c->stream);
  FinArgs f = fin_args(w, kPhaseNone);
  f.lanes_out = out;
  if (err == cudaSuccess) {
    if (dot_mode == ENPROP_DOT_CANONICAL && rows > 0) {
      err = launch_dot_tiles(s, tm, u, v, f, c->stream);
      if (err == cudaSuccess) err = launch_fin_segments(s, tm, f, c->stream);
      c->launches += 2;
    } else if (chain_aligned(u, v)) {
      err = launch_chain(s, rows, u, v, u == v ? kChainSquare : kChainProduct, f, c->stream);
      c->launches += 1;
    } else {
      err = launch_fin_serial(s, rows, u, v, f, c->stream);
      c->launches += 1;
    }
  }
  std::vector<double> h(s + 1);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(h.data(), out, (s + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(c->stream);
  if (out) cudaFree(out);
  free_work(w);
  if (err != cudaSuccess) return cuda_fail(err, "enprop_dot");
  if (lanes_host)
    for (int e = 0; e < s; ++e) lanes_host[e] = h[e];
  if (coupled_host) *coupled_host = h[s];
  return ENPROP_OK;
}

int enprop_axpby(enprop_ctx* c, int s, int64_t n, int per_lane, const double* alpha_host,
                 const double* x, const double* beta_host, double* y) {
  ScopedLaunchOpts launch_scope(c);
  if (!c || !alpha_host || !beta_host) return fail(ENPROP_ERR_INVALID, "axpby: null argument");
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  if (n == 0) return ENPROP_OK;
  std::vector<double> co(2 * s);
  for (int e = 0; e < s; ++e) {
    co[e] = per_lane ? alpha_host[e] : alpha_host[0];
    co[s + e] = per_lane ? beta_host[e] : beta_host[0];
  }
  double* d = nullptr;
  EP_CUDA(cudaMalloc(&d, 2 * s * sizeof(double)));
  cudaError_t err = cudaMemcpyAsync(d, co.data(), 2 * s * sizeof(double), cudaMemcpyHostToDevice, c->stream);
  if (err == cudaSuccess) err = launch_axpby(s, n, per_lane, d, d + s, x, y, c->stream);
  c->launches += 1;
  if (err == cudaSuccess) err = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (err != cudaSuccess) return cuda_fail(err, "enprop_axpby");
  return ENPROP_OK;
}

int enprop_cg(enprop_ctx* c, int s, int rows, const int* row_map, const int* col_entry,
              const double* values, const double* b, double* x, const enprop_cg_options* opt,
              int* iterations, int* lane_status, double* history, int* hist_len) {
  ScopedLaunchOpts launch_scope(c);
  if (!c) return fail(ENPROP_ERR_INVALID, "null context");
  int rc = validate_cg_options(opt, s);
  if (rc) return rc;
  if (rows < 0) return fail(ENPROP_ERR_INVALID, "pcg_solve: negative dimension");
  CgWork w;
  rc = run_cg(c, s, rows, row_map, col_entry, values, b, x, opt, w, iterations, lane_status,
              history, hist_len);
  free_work(w);
  return rc;
}

}  // extern "C"

// ============================================================================
// Device-resident problem (the performance path).
struct enprop_problem {
  enprop_ctx* ctx = nullptr;
  enprop_problem_desc desc{};
  int rows = 0;
  int64_t nnz = 0;
  int* row_map = nullptr;
  int* col_entry = nullptr;
  double* values = nullptr;
  double* residual = nullptr;
  double* rhs = nullptr;
  double* x = nullptr;
  double* y = nullptr;
  int* vpos = nullptr;   // symmetric storage (ENPROP_OPT_SYMMETRIC_STORAGE): slot of each entry
  int* up_start = nullptr;  // first stored slot of each row (rows + 1)
  int64_t nnz_stored = 0;
  double* u = nullptr;      // Newton iterate (enprop_problem_newton)
  StageMap stage;           // stage-pipelined CG SpMV (ep_staged.cu), built on first solve
  int stage_failed = 0;
  AsmSetup setup;
  CgWork work;
};


extern "C" {

int enprop_problem_create(enprop_ctx* c, const enprop_problem_desc* d, enprop_problem** out) {
  if (!c || !d || !out) return fail(ENPROP_ERR_INVALID, "enprop_problem_create: null argument");
  const int s = d->ensemble_size;
  if (!valid_width(s)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  const int n = d->cells_per_axis;
  if (n < 1) return fail(ENPROP_ERR_INVALID, "StructuredMesh: cells_per_axis must be at least 1");
  if (enprop_mesh_nnz(n) > 2147483647LL)
    return fail(ENPROP_ERR_INVALID, "enprop_problem_create: nnz exceeds int32");
  auto* p = new (std::nothrow) enprop_problem();
  if (!p) return fail(ENPROP_ERR_OOM, "out of host memory");
  p->ctx = c;
  p->desc = *d;
  p->rows = (n + 1) * (n + 1) * (n + 1);
  p->nnz = enprop_mesh_nnz(n);
  auto cleanup = [&](int rc) {
    enprop_problem_destroy(p);
    return rc;
  };
  int rc = make_asm_setup(c, n, &d->kl, &d->coeffs, p->setup);
  if (rc) return cleanup(rc);
  const size_t vec = (size_t)p->rows * s * sizeof(double);
  cudaError_t err;
  if ((err = cudaMalloc(&p->row_map, (p->rows + 1) * sizeof(int))) != cudaSuccess ||
      (err = cudaMalloc(&p->col_entry, p->nnz * sizeof(int))) != cudaSuccess ||
      (err = cudaMalloc(&p->residual, vec)) != cudaSuccess ||
      (err = cudaMalloc(&p->rhs, vec)) != cudaSuccess ||
      (err = cudaMalloc(&p->x, vec)) != cudaSuccess ||
      (err = cudaMalloc(&p->y, (size_t)d->kl.num_terms * s * sizeof(double))) != cudaSuccess)
    return cleanup(cuda_fail(err, "enprop_problem_create"));
  if ((err = launch_build_graph(n, p->row_map, p->col_entry, c->stream)) != cudaSuccess)
    return cleanup(cuda_fail(err, "enprop_problem_create: graph"));
  c->launches += 1;
  p->nnz_stored = p->nnz;
  // the assembled operator is exactly symmetric unless the
  // advection term (alpha != 0, fem.hpp:167-191) is on
  // symmetric storage from s = 4 up (auto): at s = 1 and 2 the slot map costs
  // about what it saves (s = 1: 28.8 MB of slots saved, 28.8 MB of slot map
  // added at 64^3) and the full-storage narrow SpMV (k_spmv_small) is faster
  // than gathering through it (64^3, s = 1: 0.077 -> 0.027 ms); at s = 8 the
  // halved value bytes win (warp kernel 0.098 ms vs 0.108 for full storage)
  if (d->coeffs.alpha == 0.0 && (c->symmetric_storage == 2 || (c->symmetric_storage == 1 && s >= 4))) {
    if ((err = cudaMalloc(&p->vpos, p->nnz * sizeof(int))) != cudaSuccess ||
        (err = cudaMalloc(&p->up_start, (p->rows + 1) * sizeof(int))) != cudaSuccess ||
        (err = build_sym(p->rows, p->row_map, p->col_entry, p->vpos, &p->nnz_stored, c->stream,
                         p->up_start)) != cudaSuccess)
      return cleanup(cuda_fail(err, "enprop_problem_create: symmetric storage"));
    c->launches += 2;
  }
  if ((err = cudaMalloc(&p->values, (size_t)p->nnz_stored * s * sizeof(double))) != cudaSuccess)
    return cleanup(cuda_fail(err, "enprop_problem_create"));
  if ((err = cudaStreamSynchronize(c->stream)) != cudaSuccess)
    return cleanup(cuda_fail(err, "enprop_problem_create"));
  *out = p;
  return ENPROP_OK;
}

int enprop_problem_destroy(enprop_problem* p) {
  if (!p) return ENPROP_OK;
  for (void* q : {(void*)p->row_map, (void*)p->col_entry, (void*)p->values, (void*)p->residual,
                  (void*)p->rhs, (void*)p->x, (void*)p->y, (void*)p->vpos, (void*)p->up_start, (void*)p->u})
    if (q) cudaFree(q);
  free_stage_map(p->stage);
  free_asm_setup(p->setup);
  free_work(p->work);
  delete p;
  return ENPROP_OK;
}

int enprop_problem_views(enprop_problem* p, int* rows, int64_t* nnz, const int** row_map,
                         const int** col_entry, double** values, double** residual,
                         double** solution) {
  if (!p) return fail(ENPROP_ERR_INVALID, "null problem");
  if (rows) *rows = p->rows;
  if (nnz) *nnz = p->nnz;
  if (row_map) *row_map = p->row_map;
  if (col_entry) *col_entry = p->col_entry;
  if (values) *values = p->values;
  if (residual) *residual = p->residual;
  if (solution) *solution = p->x;
  return ENPROP_OK;
}

int enprop_problem_storage(enprop_problem* p, int64_t* nnz_stored, const int** vpos) {
  if (!p) return fail(ENPROP_ERR_INVALID, "null problem");
  if (nnz_stored) *nnz_stored = p->nnz_stored;
  if (vpos) *vpos = p->vpos;
  return ENPROP_OK;
}

int enprop_problem_expand_values(enprop_problem* p, double* values_full) {
  if (!p || !values_full) return fail(ENPROP_ERR_INVALID, "enprop_problem_expand_values: null argument");
  const int s = p->desc.ensemble_size;
  if (!p->vpos) {
    EP_CUDA(cudaMemcpyAsync(values_full, p->values, (size_t)p->nnz * s * sizeof(double),
                            cudaMemcpyDeviceToDevice, p->ctx->stream));
  } else {
    EP_CUDA(launch_sym_expand(s, p->nnz, p->vpos, p->values, values_full, p->ctx->stream));
    p->ctx->launches += 1;
  }
  return ENPROP_OK;
}

int enprop_problem_assemble(enprop_problem* p, const double* y) {
  ScopedLaunchOpts launch_scope(p ? p->ctx : nullptr);
  if (!p || !y) return fail(ENPROP_ERR_INVALID, "enprop_problem_assemble: null argument");
  AsmArgs a = p->setup.args;
  a.u = nullptr;
  a.y = y;
  a.row_map = p->row_map;
  a.values = p->values;
  a.residual = p->residual;
  a.vpos = p->vpos;
  a.dirichlet = 1;
  a.bc0 = p->desc.bc.x0_value;
  a.bc1 = p->desc.bc.x1_value;
  EP_CUDA(launch_assemble(p->desc.ensemble_size, a, p->ctx->stream));
  p->ctx->launches += 1;
  return ENPROP_OK;
}

int enprop_problem_solve(enprop_problem* p, const enprop_cg_options* opt, int* iterations,
                         int* lane_status, double* history, int* hist_len) {
  ScopedLaunchOpts launch_scope(p ? p->ctx : nullptr);
  if (!p) return fail(ENPROP_ERR_INVALID, "null problem");
  const int s = p->desc.ensemble_size;
  int rc = validate_cg_options(opt, s);
  if (rc) return rc;
  enprop_cg_options o = *opt;
  if (o.seg_rows <= 0) o.seg_rows = (p->desc.cells_per_axis + 1) * (p->desc.cells_per_axis + 1);
  const int64_t len = (int64_t)p->rows * s;  // rhs = -residual (bench.cpp:298-299)
  EP_CUDA(launch_negate(len, p->residual, p->rhs, p->ctx->stream));
  p->ctx->launches += 1;
  // stage-pipelined SpMV (ep_staged.cu): structured graph + symmetric storage,
  // s in {4, 16, 32}, automatic variant selection; both dot orders (serial:
  // the kernel writes the p*q products for the chain kernel; its stages are
  // claimed dynamically, so SMs busy with other groups' chains do not stall it)
  const StageMap* stage = nullptr;
  const int N = p->desc.cells_per_axis + 1;
  if (p->vpos && spmv_variant() < 0 && staged_supported(s, N) && !p->stage_failed &&
      (o.dot_mode == ENPROP_DOT_CANONICAL || staged_serial())) {
    if (!p->stage.desc || p->stage.tm.seg_rows != o.seg_rows) {
      const TileMap tm = make_tile_map(p->rows, o.seg_rows);
      const cudaError_t err = build_stage_map(s, tm, N, p->row_map, p->col_entry, p->vpos,
                                              p->up_start, p->stage, p->ctx->stream);
      if (err == cudaErrorInvalidValue) {
        p->stage_failed = 1;  // not representable: the warp-per-tile kernel runs instead
        cudaGetLastError();
      } else if (err != cudaSuccess) {
        return cuda_fail(err, "enprop_problem_solve: stage map");
      } else {
        p->ctx->launches += 1;
      }
    }
    if (p->stage.desc) stage = &p->stage;
  }
  return run_cg(p->ctx, s, p->rows, p->row_map, p->col_entry, p->values, p->rhs, p->x, &o, p->work,
                iterations, lane_status, history, hist_len, p->vpos, stage);
}

}  // extern "C"

namespace {

// newton_solve (fem.hpp:265-302): mg == nullptr solves the linear systems with
// the identity preconditioner, else with MgPreconditioner of a hierarchy built
// from each step's Jacobian (the reference's own choice, :294-297).
int problem_newton(enprop_problem* p, const double* y, const enprop_newton_options* opt,
                   const enprop_mg_options* mg, int* newton_iterations, int* total_cg_iterations,
                   double* residual_norms, int* num_norms) {
  if (!p || !y || !opt) return fail(ENPROP_ERR_INVALID, "enprop_problem_newton: null argument");
  if (opt->max_iterations < 0) return fail(ENPROP_ERR_INVALID, "newton_solve: negative max_iterations");
  const int s = p->desc.ensemble_size;
  int rc = validate_cg_options(&opt->linear, s);
  if (rc) return rc;
  enprop_ctx* c = p->ctx;
  cudaStream_t st = c->stream;
  const int64_t len = (int64_t)p->rows * s;
  const size_t vec = (size_t)len * sizeof(double);
  if (!p->u) EP_CUDA(cudaMalloc(&p->u, vec));
  EP_CUDA(cudaMemsetAsync(p->u, 0, vec, st));  // result.solution = 0 (fem.hpp:271)
  const int seg = (p->desc.cells_per_axis + 1) * (p->desc.cells_per_axis + 1);
  int steps = 0, cg_total = 0, nn = 0;
  double initial = 0.0;
  double* full_vals = nullptr;  // full [nnz][s] values for the hierarchy (multigrid only)
  struct FreeOnExit {
    double*& q;
    ~FreeOnExit() {
      if (q) cudaFree(q);
    }
  } free_full{full_vals};
  auto finish = [&](int code) {
    if (newton_iterations) *newton_iterations = steps;
    if (total_cg_iterations) *total_cg_iterations = cg_total;
    if (num_norms) *num_norms = nn;
    cudaError_t err = cudaMemcpyAsync(p->x, p->u, vec, cudaMemcpyDeviceToDevice, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "enprop_problem_newton");
    return code;
  };
  for (int step = 0;; ++step) {
    AsmArgs a = p->setup.args;  // assemble at u, Dirichlet fused (fem.hpp:275-276)
    a.u = p->u;
    a.y = y;
    a.row_map = p->row_map;
    a.values = p->values;
    a.residual = p->residual;
    a.vpos = p->vpos;
    a.dirichlet = 1;
    a.bc0 = p->desc.bc.x0_value;
    a.bc1 = p->desc.bc.x1_value;
    EP_CUDA(launch_assemble(s, a, st));
    c->launches += 1;
    double dot = 0.0;  // norm2(system.residual) (fem.hpp:277), coupled
    rc = enprop_dot(c, s, len / s, p->residual, p->residual, opt->linear.dot_mode, seg, nullptr, &dot);
    if (rc) return rc;
    const double norm = std::sqrt(dot);
    if (residual_norms && nn <= opt->max_iterations) residual_norms[nn] = norm;
    ++nn;
    if (step == 0) {
      initial = norm;
      if (initial == 0.0) return finish(ENPROP_OK);
    } else if (norm < opt->tol * initial) {
      steps = step;
      return finish(ENPROP_OK);
    }
    if (step >= opt->max_iterations) {
      steps = step;
      finish(ENPROP_OK);
      return fail(ENPROP_ERR_NO_CONVERGENCE, "newton_solve: no convergence within " +
                                                 std::to_string(opt->max_iterations) + " iterations");
    }
    // rhs = -residual; J du = rhs by CG; u = 1.0*du + 1.0*u (fem.hpp:294-300)
    const int lanes = opt->linear.flavour == ENPROP_CG_UNCOUPLED ? s : 1;
    std::vector<int> its(lanes, 0), ls(lanes, 0);
    if (mg) {  // build_hierarchy(system.matrix) + pcg_solve(..., MgPreconditioner) (:294-297)
      if (opt->linear.dot_mode != ENPROP_DOT_SERIAL)
        return fail(ENPROP_ERR_INVALID, "newton_solve (multigrid): the reference's serial dot order only");
      if (!full_vals) EP_CUDA(cudaMalloc(&full_vals, (size_t)p->nnz * s * sizeof(double)));
      rc = enprop_problem_expand_values(p, full_vals);
      if (rc) return rc;
      EP_CUDA(launch_negate(len, p->residual, p->rhs, st));
      c->launches += 1;
      enprop_mg* h = nullptr;
      rc = enprop_mg_build(c, s, p->rows, p->row_map, p->col_entry, full_vals, mg, &h);
      if (rc) return rc;
      rc = enprop_mg_pcg(h, p->rhs, p->x, &opt->linear, its.data(), ls.data(), nullptr, nullptr);
      const std::string msg = rc ? g_last_error : std::string();
      enprop_mg_destroy(h);
      if (rc) g_last_error = msg;
    } else {
      rc = enprop_problem_solve(p, &opt->linear, its.data(), ls.data(), nullptr, nullptr);
    }
    int mx = 0;
    for (int l = 0; l < lanes; ++l) mx = its[l] > mx ? its[l] : mx;
    cg_total += mx;
    if (rc) {
      steps = step;
      const std::string msg = g_last_error;
      finish(ENPROP_OK);
      return fail(rc, msg);
    }
    const double one = 1.0;
    rc = enprop_axpby(c, s, len / s, 0, &one, p->x, &one, p->u);
    if (rc) return rc;
  }
}

}  // namespace

extern "C" {

int enprop_problem_newton(enprop_problem* p, const double* y, const enprop_newton_options* opt,
                          int* newton_iterations, int* total_cg_iterations, double* residual_norms,
                          int* num_norms) {
  ScopedLaunchOpts launch_scope(p ? p->ctx : nullptr);
  return problem_newton(p, y, opt, nullptr, newton_iterations, total_cg_iterations, residual_norms, num_norms);
}

int enprop_problem_newton_mg(enprop_problem* p, const double* y, const enprop_newton_options* opt,
                             const enprop_mg_options* mg, int* newton_iterations, int* total_cg_iterations,
                             double* residual_norms, int* num_norms) {
  ScopedLaunchOpts launch_scope(p ? p->ctx : nullptr);
  enprop_mg_options d{500, 2, 30.0, 1.1, 40};  // MgOptions defaults (multigrid.hpp:14-20)
  return problem_newton(p, y, opt, mg ? mg : &d, newton_iterations, total_cg_iterations, residual_norms,
                        num_norms);
}

int enprop_problem_solve_host(enprop_problem* p, const double* y_host, double* x_host,
                              const enprop_cg_options* opt, int* iterations, int* lane_status) {
  ScopedLaunchOpts launch_scope(p ? p->ctx : nullptr);
  if (!p || !y_host || !x_host) return fail(ENPROP_ERR_INVALID, "enprop_problem_solve_host: null argument");
  const int s = p->desc.ensemble_size;
  cudaStream_t st = p->ctx->stream;
  EP_CUDA(cudaMemcpyAsync(p->y, y_host, (size_t)p->desc.kl.num_terms * s * sizeof(double),
                          cudaMemcpyHostToDevice, st));
  int rc = enprop_problem_assemble(p, p->y);
  if (rc) return rc;
  rc = enprop_problem_solve(p, opt, iterations, lane_status, nullptr, nullptr);
  if (rc && rc != ENPROP_ERR_NO_CONVERGENCE && rc != ENPROP_ERR_INDEFINITE) return rc;
  EP_CUDA(cudaMemcpyAsync(x_host, p->x, (size_t)p->rows * s * sizeof(double), cudaMemcpyDeviceToHost, st));
  EP_CUDA(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"

namespace ep_internal {
__global__ void k_negate(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = -a[i];
}
cudaError_t launch_negate(int64_t n, const double* a, double* b, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_negate<<<(int)((n + 255) / 256), 256, 0, st>>>(n, a, b);
  return cudaGetLastError();
}
}  // namespace ep_internal
