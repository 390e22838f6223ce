// Multi-GPU ensemble solve by 1-D slab decomposition of the node planes.
//
// Decomposition (the reference's partition.cpp:31-72 rule applied to z-planes
// of nodes: lower ranks take the extra plane). With x-fastest numbering
// (mesh.hpp:24-26) a z-slab is a contiguous row range, so a rank's matrix is a
// slice of the global CRS and a ghost plane is one contiguous N^2 * s block:
//   owned rows   [k0 N^2, k1 N^2)
//   ext layout   [lo ghost plane | owned planes | hi ghost plane]  (gathered p)
// Assembly needs no communication (node-centric gather over the cells around
// each owned node). Per CG iteration: direction pass -> halo of p_new (one
// plane to each neighbour) -> SpMV with p.q per-plane sums -> all-gather of
// the per-plane sums -> canonical total in global plane order -> update ->
// all-gather -> total. The canonical order makes every rank's
// totals, hence alpha/beta/iterations/solutions, identical to the one-GPU
// solve bit for bit, independent of the rank count.
//
// Transports:
//  * NCCL (one process per GPU; libnccl.so.2 loaded at run time, so an already
//    loaded copy -- e.g. torch's -- is shared): ncclSend/ncclRecv for the halo,
//    ncclAllGather for the per-plane sums;
//  * CUDA IPC (one process per rank, any GPUs of one node, including several
//    ranks on ONE GPU, which NCCL refuses): every rank exports its p buffers,
//    its per-plane sum buffers and three interprocess events; a host board in
//    /dev/shm carries the handles and, per rank and event kind, how many
//    records have been issued. A consumer waits on the host until the
//    producer's record for the needed step has been issued, then makes its
//    stream wait on the producer's event (cudaStreamWaitEvent) and copies from
//    the peer's memory with cudaMemcpyAsync (NVLink P2P between GPUs, a device
//    copy on one GPU). No kernel ever waits on another rank: only stream-event
//    waits, so co-located ranks cannot deadlock each other's SMs.
//    Ordering: halo pulls and all-gathers happen every phase, so no rank can
//    issue the next record of a kind before every peer has issued its wait on
//    the current one (each record follows the rank's waits on all peers'
//    previous phase); the per-plane sums are double buffered by phase (p.q /
//    r.r) so a fast rank never overwrites sums a slow rank still copies;
//  * an in-process emulation of all ranks on one GPU where the halo and the
//    all-gather are stream-ordered device copies (testing).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "enprop_b200.h"
#include "ep_internal.h"
#include "ep_kernels.h"

using namespace ep;
using namespace ep_internal;

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
#define EP_SYM(f, name)                                             \
  f = reinterpret_cast<decltype(f)>(dlsym(h, name));                \
  if (!f) return false;
    EP_SYM(GetUniqueId, "ncclGetUniqueId");
    EP_SYM(CommInitRank, "ncclCommInitRank");
    EP_SYM(CommDestroy, "ncclCommDestroy");
    EP_SYM(Send, "ncclSend");
    EP_SYM(Recv, "ncclRecv");
    EP_SYM(GroupStart, "ncclGroupStart");
    EP_SYM(GroupEnd, "ncclGroupEnd");
    EP_SYM(AllGather, "ncclAllGather");
    EP_SYM(GetErrorString, "ncclGetErrorString");
#undef EP_SYM
    return true;
  }
};

NcclApi& nccl() {
  static NcclApi api;
  return api;
}

#define EP_NCCL(call)                                                                   \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess)                                                              \
      return fail(ENPROP_ERR_CUDA, std::string(#call) + ": " + nccl().GetErrorString(_r)); \
  } while (0)

// start of global row g in the 27-point graph (closed form, as k_build_graph)
int64_t graph_start(int n, int64_t g) {
  const int64_t N = n + 1, W = 3 * N - 2;
  auto cnt = [N](int64_t t) { return 1 + (t > 0) + (t < N - 1); };
  auto pre = [](int64_t t) { return t == 0 ? 0 : 2 + 3 * (t - 1); };
  const int64_t i = g % N, j = (g / N) % N, k = g / (N * N);
  if (g >= N * N * N) return (3 * N - 2) * (3 * N - 2) * (3 * N - 2);
  return pre(k) * W * W + cnt(k) * (pre(j) * W + cnt(j) * pre(i));
}

// One rank's slab: graph slice, matrix, CG vectors (p in ext layout).
struct DistRank {
  int rank = 0, k0 = 0, k1 = 0;
  int row_begin = 0, rows = 0, lo_rows = 0, hi_rows = 0, ext_begin = 0;
  int64_t nnz = 0;
  int* row_map = nullptr;
  int* col_entry = nullptr;
  double *values = nullptr, *residual = nullptr, *x = nullptr, *r = nullptr, *q = nullptr;
  double* p[2] = {nullptr, nullptr};  // ext layout
  TileMap tm{};
  double *partials = nullptr, *gathered = nullptr, *hist = nullptr;
  // per-plane sums of this rank: [0] init r.r and p.q, [1] r.r and Newton's
  // residual norm; see seg_buffer for why the phases alternate this way
  double* seg[2] = {nullptr, nullptr};
  int* counters = nullptr;
  int* plane_pos = nullptr;
  CgState* state = nullptr;
  double* u = nullptr;  // Newton iterate, owned rows (enprop_dist_newton)
  // staged mode (s in {4, 16, 32}, alpha = 0): symmetric storage of the store
  // rows = lo ghost plane + owned rows (the ghost plane's upper slots are
  // assembled here, no communication) and the stage-pipelined SpMV in owned
  // coordinates (columns of the store graph are owned-row coordinates; the x
  // runs reach the ghost planes of the ext p buffer)
  bool staged = false;
  int store_rows = 0;
  int* vpos = nullptr;
  int* up_start = nullptr;
  int64_t nnz_stored = 0;
  StageMap stage;
};

}  // namespace

namespace {
enum Transport { kEmulated = 0, kNccl = 1, kIpc = 2 };
enum EvKind { kEvP = 0, kEvPQ = 1, kEvRR = 2, kEvSync = 3, kEvKinds = 4 };
constexpr int kIpcMaxRanks = 64;

// Host board of an IPC job (/dev/shm, one per job name, zero-filled on creation).
struct IpcSlot {
  cudaIpcMemHandle_t p[2], seg[2];
  cudaIpcEventHandle_t ev[kEvKinds];
  int device;
  std::atomic<int> published;
  std::atomic<long long> seq[kEvKinds];  // records issued per event kind
};
struct IpcBoard {
  std::atomic<int> joined, opened, closed;
  IpcSlot slot[kIpcMaxRanks];
};
}  // namespace

struct enprop_dist {
  enprop_ctx* ctx = nullptr;
  enprop_problem_desc desc{};
  int nranks = 1, n = 0, N = 0, plane = 0, maxplanes = 0, maxit = -1;
  int transport = kEmulated;
  bool emulated = true;
  ncclComm_t comm = nullptr;
  AsmSetup setup;
  std::vector<DistRank> ranks;  // emulated: all ranks; NCCL / IPC: this process's rank
  // halo overlap: the halo runs on `side` while the interior stages run
  cudaStream_t side = nullptr;
  cudaEvent_t ev_owned = nullptr, ev_halo = nullptr;
  // IPC transport
  std::string board_name;
  IpcBoard* board = nullptr;
  cudaEvent_t ev[kEvKinds] = {};
  long long seq[kEvKinds] = {};
  std::vector<double*> peer_p[2], peer_seg[2];  // opened peer buffers (own ones for self)
  std::vector<cudaEvent_t> peer_ev[kEvKinds];
  bool ipc_open = false;
};

namespace {

void plane_range(int N, int P, int r, int& k0, int& k1) {
  const int base = N / P, extra = N % P;  // partition.cpp:50-58
  k0 = r * base + std::min(r, extra);
  k1 = k0 + base + (r < extra ? 1 : 0);
}

void free_rank(DistRank& d) {
  for (void* q : {(void*)d.row_map, (void*)d.col_entry, (void*)d.values, (void*)d.residual,
                  (void*)d.x, (void*)d.r, (void*)d.q, (void*)d.p[0], (void*)d.p[1],
                  (void*)d.partials, (void*)d.seg[0], (void*)d.seg[1], (void*)d.gathered, (void*)d.hist,
                  (void*)d.counters, (void*)d.plane_pos, (void*)d.state, (void*)d.vpos, (void*)d.up_start, (void*)d.u})
    if (q) cudaFree(q);
  free_stage_map(d.stage);
  d = DistRank{};
}

int setup_rank(enprop_dist* D, DistRank& d, int r) {
  const int s = D->desc.ensemble_size;
  const int n = D->n, N = D->N, plane = D->plane, P = D->nranks;
  d.rank = r;
  plane_range(N, P, r, d.k0, d.k1);
  d.row_begin = d.k0 * plane;
  d.rows = (d.k1 - d.k0) * plane;
  d.lo_rows = d.k0 > 0 ? plane : 0;
  d.hi_rows = d.k1 < N ? plane : 0;
  d.ext_begin = d.row_begin - d.lo_rows;
  d.staged = staged_supported(s, N) && D->desc.coeffs.alpha == 0.0 && D->ctx->symmetric_storage != 0;
  d.store_rows = d.staged ? d.lo_rows + d.rows : d.rows;
  const int store_begin = d.row_begin + d.rows - d.store_rows;  // ext_begin when staged
  d.nnz = graph_start(n, d.row_begin + d.rows) - graph_start(n, store_begin);
  const size_t vec = (size_t)d.rows * s * sizeof(double);
  const size_t ext = (size_t)(d.lo_rows + d.rows + d.hi_rows) * s * sizeof(double);
  d.tm = make_tile_map(d.rows, plane);
  EP_CUDA(cudaMalloc(&d.row_map, (d.store_rows + 1) * sizeof(int)));
  EP_CUDA(cudaMalloc(&d.col_entry, d.nnz * sizeof(int)));
  EP_CUDA(cudaMalloc(&d.residual, (size_t)d.store_rows * s * sizeof(double)));
  EP_CUDA(cudaMalloc(&d.x, vec));
  EP_CUDA(cudaMalloc(&d.r, vec));
  EP_CUDA(cudaMalloc(&d.q, vec));
  EP_CUDA(cudaMalloc(&d.p[0], ext));
  EP_CUDA(cudaMalloc(&d.p[1], ext));
  EP_CUDA(cudaMemset(d.p[0], 0, ext));
  EP_CUDA(cudaMemset(d.p[1], 0, ext));
  EP_CUDA(cudaMalloc(&d.partials, (size_t)std::max(d.tm.num_tiles(), 1) * s * sizeof(double)));
  for (int k = 0; k < 2; ++k) {
    EP_CUDA(cudaMalloc(&d.seg[k], (size_t)D->maxplanes * s * sizeof(double)));
    EP_CUDA(cudaMemset(d.seg[k], 0, (size_t)D->maxplanes * s * sizeof(double)));
  }
  EP_CUDA(cudaMalloc(&d.gathered, (size_t)P * D->maxplanes * s * sizeof(double)));
  EP_CUDA(cudaMalloc(&d.counters, kCounterInts * sizeof(int)));
  EP_CUDA(cudaMemset(d.counters, 0, kCounterInts * sizeof(int)));
  EP_CUDA(cudaMalloc(&d.state, sizeof(CgState)));
  // global plane k lives at gathered[rank_of(k) * maxplanes + (k - k0(rank))]
  std::vector<int> pos(N);
  for (int q = 0; q < P; ++q) {
    int a, b;
    plane_range(N, P, q, a, b);
    for (int k = a; k < b; ++k) pos[k] = q * D->maxplanes + (k - a);
  }
  EP_CUDA(cudaMalloc(&d.plane_pos, N * sizeof(int)));
  EP_CUDA(cudaMemcpy(d.plane_pos, pos.data(), N * sizeof(int), cudaMemcpyHostToDevice));
  cudaStream_t st = D->ctx->stream;
  if (!d.staged) {  // full storage, columns in ext-buffer coordinates (the warp SpMV reads p from 0)
    EP_CUDA(launch_build_graph_range(n, d.row_begin, d.rows, d.ext_begin, d.row_map, d.col_entry, st));
    EP_CUDA(cudaMalloc(&d.values, (size_t)d.nnz * s * sizeof(double)));
    d.nnz_stored = d.nnz;
    D->ctx->launches += 1;
    return ENPROP_OK;
  }
  // store rows [ext_begin, row_begin + rows), columns in owned coordinates
  EP_CUDA(launch_build_graph_range(n, store_begin, d.store_rows, d.row_begin, d.row_map, d.col_entry, st));
  EP_CUDA(cudaMalloc(&d.vpos, d.nnz * sizeof(int)));
  EP_CUDA(cudaMalloc(&d.up_start, (d.store_rows + 1) * sizeof(int)));
  EP_CUDA(build_sym(d.store_rows, d.row_map, d.col_entry, d.vpos, &d.nnz_stored, st, d.up_start, d.lo_rows));
  EP_CUDA(cudaMalloc(&d.values, (size_t)d.nnz_stored * s * sizeof(double)));
  // interior stages: rows at least one plane away from every ghost plane
  // (ranks with a neighbour; ENPROP_DIST_OVERLAP=0 keeps one launch, A/B)
  const bool split = (d.lo_rows || d.hi_rows) && env_int("ENPROP_DIST_OVERLAP", 1) != 0;
  const int ilo = split ? (d.lo_rows ? plane : 0) : 0, ihi = split ? (d.hi_rows ? d.rows - plane : d.rows) : 0;
  EP_CUDA(build_stage_map(s, d.tm, N, d.row_map + d.lo_rows, d.col_entry, d.vpos, d.up_start + d.lo_rows,
                          d.stage, st, -d.lo_rows, d.rows + d.hi_rows, ilo, ihi));
  D->ctx->launches += 4;
  return ENPROP_OK;
}

// Which per-plane sum buffer a phase writes. Over IPC a peer pulls this
// rank's buffer on its own stream after this rank publishes it. The pull is
// known complete only once that peer publishes again and this rank's stream
// waits on it. The all-gathers wait on every rank, so alternating buffers
// orders the CG loop: init (1), PQ (0), RR (1), PQ (0), ... Newton's norm (0)
// follows a solve's last RR, which waited on every rank's publish after its
// last PQ pull. A solve's init follows the last RR of the previous solve on the
// same buffer, and ipc_quiesce orders that (halos order only the neighbours).
int seg_buffer(int phase) { return phase == kPhasePQ || phase == kPhaseNone ? 0 : 1; }

FinArgs rank_fin(const DistRank& d, int phase) {
  FinArgs f;
  f.partials = d.partials;
  f.seg_sums = d.seg[seg_buffer(phase)];
  f.seg_done = d.counters;
  f.bar = d.counters + 1;
  f.ticket = d.counters + 3;
  f.prod = nullptr;
  f.phase = phase;
  f.cg = d.state;
  f.hist = d.hist;
  f.lanes_out = nullptr;
  f.seg_only = 1;
  f.defer = 1;
  return f;
}

// owned-row layout of rank r: (ext_begin, lo ghost rows, owned rows)
void rank_layout(const enprop_dist* D, int r, int& ext_begin, int& lo_rows, int& rows) {
  int k0, k1;
  plane_range(D->N, D->nranks, r, k0, k1);
  lo_rows = k0 > 0 ? D->plane : 0;
  rows = (k1 - k0) * D->plane;
  ext_begin = k0 * D->plane - lo_rows;
}

constexpr double kIpcTimeoutS = 120.0;

// host wait until rank q has issued `target` records of `kind` (or time out)
int ipc_wait_seq(enprop_dist* D, int q, int kind, long long target) {
  auto& cnt = D->board->slot[q].seq[kind];
  if (cnt.load(std::memory_order_acquire) >= target) return ENPROP_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0; cnt.load(std::memory_order_acquire) < target; ++spin) {
    if ((spin & 1023) == 1023) {
      sched_yield();
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kIpcTimeoutS)
        return fail(ENPROP_ERR_CUDA, "enprop_dist (ipc): timed out waiting for rank " + std::to_string(q));
    }
  }
  return ENPROP_OK;
}

// record this rank's event of `kind` after the work already on the stream and
// announce it on the board
int ipc_publish(enprop_dist* D, int kind) {
  EP_CUDA(cudaEventRecord(D->ev[kind], D->ctx->stream));
  D->seq[kind] += 1;
  D->board->slot[D->ranks[0].rank].seq[kind].store(D->seq[kind], std::memory_order_release);
  return ENPROP_OK;
}

// make stream `st` (default: the context's) wait for rank q's record of `kind` matching ours
int ipc_wait(enprop_dist* D, int q, int kind, cudaStream_t st = nullptr) {
  int rc = ipc_wait_seq(D, q, kind, D->seq[kind]);
  if (rc) return rc;
  EP_CUDA(cudaStreamWaitEvent(st ? st : D->ctx->stream, D->peer_ev[kind][q], 0));
  return ENPROP_OK;
}

// device-side all-rank fence: this stream continues once every rank's stream
// has reached its own ipc_quiesce (and so finished its earlier pulls)
int ipc_quiesce(enprop_dist* D) {
  int rc = ipc_publish(D, kEvSync);
  for (int q = 0; q < D->nranks && !rc; ++q)
    if (q != D->ranks[0].rank) rc = ipc_wait(D, q, kEvSync);
  return rc;
}

// wait on the host until every rank has bumped `counter` to nranks
int ipc_barrier(enprop_dist* D, std::atomic<int>& counter) {
  counter.fetch_add(1, std::memory_order_acq_rel);
  const auto t0 = std::chrono::steady_clock::now();
  while (counter.load(std::memory_order_acquire) < D->nranks) {
    sched_yield();
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kIpcTimeoutS)
      return fail(ENPROP_ERR_CUDA, "enprop_dist (ipc): timed out waiting for the other ranks to join");
  }
  return ENPROP_OK;
}

int ipc_setup(enprop_dist* D, const char* job) {
  D->board_name = std::string("/enprop_b200_") + job;
  const int fd = shm_open(D->board_name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) return fail(ENPROP_ERR_CUDA, "enprop_dist (ipc): shm_open failed for " + D->board_name);
  if (ftruncate(fd, sizeof(IpcBoard)) != 0) {
    close(fd);
    return fail(ENPROP_ERR_CUDA, "enprop_dist (ipc): ftruncate failed");
  }
  void* m = mmap(nullptr, sizeof(IpcBoard), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) return fail(ENPROP_ERR_CUDA, "enprop_dist (ipc): mmap failed");
  D->board = static_cast<IpcBoard*>(m);
  DistRank& d = D->ranks[0];
  IpcSlot& me = D->board->slot[d.rank];
  for (int k = 0; k < kEvKinds; ++k) {
    EP_CUDA(cudaEventCreateWithFlags(&D->ev[k], cudaEventDisableTiming | cudaEventInterprocess));
    EP_CUDA(cudaIpcGetEventHandle(&me.ev[k], D->ev[k]));
  }
  for (int k = 0; k < 2; ++k) {
    EP_CUDA(cudaIpcGetMemHandle(&me.p[k], d.p[k]));
    EP_CUDA(cudaIpcGetMemHandle(&me.seg[k], d.seg[k]));
  }
  EP_CUDA(cudaGetDevice(&me.device));
  me.published.store(1, std::memory_order_release);
  int rc = ipc_barrier(D, D->board->joined);
  if (rc) return rc;
  for (int k = 0; k < 2; ++k) {
    D->peer_p[k].assign(D->nranks, nullptr);
    D->peer_seg[k].assign(D->nranks, nullptr);
  }
  for (int k = 0; k < kEvKinds; ++k) D->peer_ev[k].assign(D->nranks, nullptr);
  D->ipc_open = true;
  for (int q = 0; q < D->nranks; ++q) {
    IpcSlot& sl = D->board->slot[q];
    const bool self = q == d.rank;
    const bool nb = q == d.rank - 1 || q == d.rank + 1;
    for (int k = 0; k < 2; ++k) {
      if (self) {
        D->peer_p[k][q] = d.p[k];
        D->peer_seg[k][q] = d.seg[k];
        continue;
      }
      void* ptr = nullptr;
      if (nb) {
        EP_CUDA(cudaIpcOpenMemHandle(&ptr, sl.p[k], cudaIpcMemLazyEnablePeerAccess));
        D->peer_p[k][q] = static_cast<double*>(ptr);
      }
      EP_CUDA(cudaIpcOpenMemHandle(&ptr, sl.seg[k], cudaIpcMemLazyEnablePeerAccess));
      D->peer_seg[k][q] = static_cast<double*>(ptr);
    }
    for (int k = 0; k < kEvKinds; ++k) {
      if (self) D->peer_ev[k][q] = D->ev[k];
      else EP_CUDA(cudaIpcOpenEventHandle(&D->peer_ev[k][q], sl.ev[k]));
    }
  }
  return ipc_barrier(D, D->board->opened);
}

void ipc_teardown(enprop_dist* D) {
  if (!D->board) return;
  const int me = D->ranks.empty() ? -1 : D->ranks[0].rank;
  if (D->ipc_open) {
    cudaStreamSynchronize(D->ctx->stream);
    for (int q = 0; q < D->nranks; ++q) {
      if (q == me) continue;
      for (int k = 0; k < 2; ++k) {
        if (D->peer_p[k][q]) cudaIpcCloseMemHandle(D->peer_p[k][q]);
        if (D->peer_seg[k][q]) cudaIpcCloseMemHandle(D->peer_seg[k][q]);
      }
    }
  }
  // the last rank out removes the board; peers keep their exported buffers
  // alive until everyone has closed its mappings
  ipc_barrier(D, D->board->closed);
  for (int k = 0; k < kEvKinds; ++k)
    if (D->ev[k]) cudaEventDestroy(D->ev[k]);
  if (me == 0) shm_unlink(D->board_name.c_str());
  munmap(D->board, sizeof(IpcBoard));
  D->board = nullptr;
}

// halo of the p buffer `which` (first owned plane -> rank-1's hi ghost, last
// owned plane -> rank+1's lo ghost), its copies on stream `st` (default: the
// context's); the owned planes must be complete on the context's stream
// (IPC: publish = false when the caller already published the owned planes)
int halo(enprop_dist* D, int which, cudaStream_t st = nullptr, bool publish = true) {
  const int s = D->desc.ensemble_size;
  const size_t pe = (size_t)D->plane * s;
  if (!st) st = D->ctx->stream;
  if (D->emulated) {
    for (size_t i = 0; i < D->ranks.size(); ++i) {
      DistRank& d = D->ranks[i];
      if (i > 0) {
        DistRank& lo = D->ranks[i - 1];
        EP_CUDA(cudaMemcpyAsync(lo.p[which] + (size_t)(lo.lo_rows + lo.rows) * s, d.p[which] + (size_t)d.lo_rows * s,
                                pe * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
      if (i + 1 < D->ranks.size()) {
        DistRank& hi = D->ranks[i + 1];
        EP_CUDA(cudaMemcpyAsync(hi.p[which], d.p[which] + (size_t)(d.lo_rows + d.rows - D->plane) * s,
                                pe * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
    }
    return ENPROP_OK;
  }
  DistRank& d = D->ranks[0];
  if (D->transport == kIpc) {  // publish p[which], pull the neighbours' boundary planes
    int rc = publish ? ipc_publish(D, kEvP) : ENPROP_OK;
    if (rc) return rc;
    if (d.rank > 0) {
      int lo, lr, rws;
      rank_layout(D, d.rank - 1, lo, lr, rws);
      if ((rc = ipc_wait(D, d.rank - 1, kEvP, st))) return rc;
      EP_CUDA(cudaMemcpyAsync(d.p[which], D->peer_p[which][d.rank - 1] + (size_t)(lr + rws - D->plane) * s,
                              pe * sizeof(double), cudaMemcpyDefault, st));
    }
    if (d.rank + 1 < D->nranks) {
      int lo, lr, rws;
      rank_layout(D, d.rank + 1, lo, lr, rws);
      if ((rc = ipc_wait(D, d.rank + 1, kEvP, st))) return rc;
      EP_CUDA(cudaMemcpyAsync(d.p[which] + (size_t)(d.lo_rows + d.rows) * s, D->peer_p[which][d.rank + 1] + (size_t)lr * s,
                              pe * sizeof(double), cudaMemcpyDefault, st));
    }
    return ENPROP_OK;
  }
  auto& api = nccl();
  EP_NCCL(api.GroupStart());
  if (d.rank > 0) {
    EP_NCCL(api.Send(d.p[which] + (size_t)d.lo_rows * s, pe, ncclDouble, d.rank - 1, D->comm, st));
    EP_NCCL(api.Recv(d.p[which], pe, ncclDouble, d.rank - 1, D->comm, st));
  }
  if (d.rank + 1 < D->nranks) {
    EP_NCCL(api.Send(d.p[which] + (size_t)(d.lo_rows + d.rows - D->plane) * s, pe, ncclDouble, d.rank + 1, D->comm, st));
    EP_NCCL(api.Recv(d.p[which] + (size_t)(d.lo_rows + d.rows) * s, pe, ncclDouble, d.rank + 1, D->comm, st));
  }
  EP_NCCL(api.GroupEnd());
  return ENPROP_OK;
}

// all-gather of the per-plane sums of `phase` (buffer seg_buffer(phase))
int allgather(enprop_dist* D, int phase) {
  const size_t cnt = (size_t)D->maxplanes * D->desc.ensemble_size;
  const int b = seg_buffer(phase);
  cudaStream_t st = D->ctx->stream;
  if (D->emulated) {
    for (auto& dst : D->ranks)
      for (size_t q = 0; q < D->ranks.size(); ++q)
        EP_CUDA(cudaMemcpyAsync(dst.gathered + q * cnt, D->ranks[q].seg[b], cnt * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    return ENPROP_OK;
  }
  DistRank& d = D->ranks[0];
  if (D->transport == kIpc) {
    const int kind = phase == kPhasePQ ? kEvPQ : kEvRR;
    int rc = ipc_publish(D, kind);
    if (rc) return rc;
    for (int q = 0; q < D->nranks; ++q) {
      if (q != d.rank && (rc = ipc_wait(D, q, kind))) return rc;
      EP_CUDA(cudaMemcpyAsync(d.gathered + q * cnt, D->peer_seg[b][q], cnt * sizeof(double), cudaMemcpyDefault, st));
    }
    return ENPROP_OK;
  }
  EP_NCCL(nccl().AllGather(d.seg[b], d.gathered, cnt, ncclDouble, D->comm, st));
  return ENPROP_OK;
}

int fin_all(enprop_dist* D, int phase, double* lanes_out = nullptr) {
  const int s = D->desc.ensemble_size;
  for (auto& d : D->ranks) {
    EP_CUDA(launch_fin_gathered(s, D->N, d.gathered, d.plane_pos, phase, d.state, d.hist, lanes_out,
                                D->ctx->stream));
    D->ctx->launches += 1;
  }
  return ENPROP_OK;
}

}  // namespace

extern "C" {

int enprop_nccl_unique_id(void* out, size_t bytes) {
  if (!out || bytes < sizeof(ncclUniqueId)) return fail(ENPROP_ERR_INVALID, "enprop_nccl_unique_id: buffer too small");
  if (!nccl().load()) return fail(ENPROP_ERR_CUDA, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  EP_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return ENPROP_OK;
}

int enprop_dist_destroy(enprop_dist* D) {
  if (!D) return ENPROP_OK;
  ipc_teardown(D);
  for (auto& d : D->ranks) free_rank(d);
  if (D->side) cudaStreamDestroy(D->side);
  if (D->ev_owned) cudaEventDestroy(D->ev_owned);
  if (D->ev_halo) cudaEventDestroy(D->ev_halo);
  free_asm_setup(D->setup);
  if (D->comm) nccl().CommDestroy(D->comm);
  delete D;
  return ENPROP_OK;
}

static int dist_create(enprop_ctx* c, const enprop_problem_desc* desc, int nranks, int rank,
                       const void* nccl_id, const char* ipc_job, enprop_dist** out) {
  if (!c || !desc || !out) return fail(ENPROP_ERR_INVALID, "enprop_dist_create: null argument");
  if (!valid_width(desc->ensemble_size)) return fail(ENPROP_ERR_INVALID, "ensemble width outside {1,2,4,8,16,32}");
  const int n = desc->cells_per_axis;
  if (n < 1) return fail(ENPROP_ERR_INVALID, "StructuredMesh: cells_per_axis must be at least 1");
  if (nranks < 1 || nranks > n + 1)  // partition.cpp:35-38
    return fail(ENPROP_ERR_INVALID, "partition: ranks must be in [1, node planes]");
  if (rank < 0 || rank >= nranks) return fail(ENPROP_ERR_INVALID, "enprop_dist_create: bad rank");
  auto* D = new (std::nothrow) enprop_dist();
  if (!D) return fail(ENPROP_ERR_OOM, "out of host memory");
  D->ctx = c;
  D->desc = *desc;
  D->nranks = nranks;
  D->n = n;
  D->N = n + 1;
  D->plane = D->N * D->N;
  D->maxplanes = (D->N + nranks - 1) / nranks;
  D->transport = nccl_id ? kNccl : (ipc_job ? kIpc : kEmulated);
  D->emulated = D->transport == kEmulated;
  auto bail = [&](int rc) {
    enprop_dist_destroy(D);
    return rc;
  };
  int rc = make_asm_setup(c, n, &desc->kl, &desc->coeffs, D->setup);
  if (rc) return bail(rc);
  if (cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&D->ev_owned, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&D->ev_halo, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(ENPROP_ERR_CUDA, "enprop_dist_create: stream / event creation failed"));
  if (D->transport == kNccl) {
    if (!nccl().load()) return bail(fail(ENPROP_ERR_CUDA, "libnccl.so.2 could not be loaded"));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = nccl().CommInitRank(&D->comm, nranks, id, rank);
    if (r != ncclSuccess) return bail(fail(ENPROP_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r)));
  }
  const int local = D->emulated ? nranks : 1;
  D->ranks.resize(local);
  for (int i = 0; i < local; ++i) {
    rc = setup_rank(D, D->ranks[i], D->emulated ? i : rank);
    if (rc) return bail(rc);
  }
  cudaError_t err = cudaStreamSynchronize(c->stream);
  if (err != cudaSuccess) return bail(cuda_fail(err, "enprop_dist_create"));
  if (D->transport == kIpc) {
    if (nranks > kIpcMaxRanks) return bail(fail(ENPROP_ERR_INVALID, "enprop_dist (ipc): at most 64 ranks"));
    rc = ipc_setup(D, ipc_job);
    if (rc) return bail(rc);
  }
  *out = D;
  return ENPROP_OK;
}

int enprop_dist_create(enprop_ctx* c, const enprop_problem_desc* desc, int nranks, int rank,
                       const void* nccl_id, enprop_dist** out) {
  return dist_create(c, desc, nranks, rank, nccl_id, nullptr, out);
}

int enprop_dist_create_ipc(enprop_ctx* c, const enprop_problem_desc* desc, int nranks, int rank,
                           const char* job, enprop_dist** out) {
  if (!job || !*job || std::strchr(job, '/'))
    return fail(ENPROP_ERR_INVALID, "enprop_dist_create_ipc: job name must be non-empty, without '/'");
  return dist_create(c, desc, nranks, rank, nullptr, job, out);
}

int enprop_dist_time_halo(enprop_dist* D, int reps, double* seconds) {
  if (!D || !seconds || reps < 1) return fail(ENPROP_ERR_INVALID, "enprop_dist_time_halo: bad argument");
  cudaStream_t st = D->ctx->stream;
  cudaEvent_t e0, e1;
  EP_CUDA(cudaEventCreate(&e0));
  EP_CUDA(cudaEventCreate(&e1));
  int rc = halo(D, 0);  // warm-up (NCCL connection setup)
  if (!rc) {
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps && !rc; ++i) rc = halo(D, 0);
    cudaEventRecord(e1, st);
  }
  float ms = 0.0f;
  cudaError_t err = cudaEventSynchronize(e1);
  if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  if (err != cudaSuccess) return cuda_fail(err, "enprop_dist_time_halo");
  *seconds = (double)ms / 1e3 / reps;
  return ENPROP_OK;
}

int enprop_write_exchange_trace_csv(const char* path, const enprop_exchange_record* recs, int count) {
  // halo.cpp:192-202, same format
  if (!path || count < 0 || (count > 0 && !recs))
    return fail(ENPROP_ERR_INVALID, "write_exchange_trace_csv: bad argument");
  std::FILE* f = std::fopen(path, "w");
  if (f == nullptr) return fail(ENPROP_ERR_INVALID, std::string("write_exchange_trace_csv: cannot open ") + path);
  std::fputs("rank,neighbor,bytes,virtual_time\n", f);
  for (int i = 0; i < count; ++i)
    std::fprintf(f, "%d,%d,%lld,%.17g\n", recs[i].rank, recs[i].neighbor, static_cast<long long>(recs[i].bytes),
                 recs[i].time);
  if (std::fclose(f) != 0)
    return fail(ENPROP_ERR_INVALID, std::string("write_exchange_trace_csv: failed writing ") + path);
  return ENPROP_OK;
}

int enprop_dist_exchange_trace(enprop_dist* D, enprop_exchange_record* out, int max_records, int* count,
                               double* elapsed_seconds) {
  if (!D || !count) return fail(ENPROP_ERR_INVALID, "enprop_dist_exchange_trace: null argument");
  const int s = D->desc.ensemble_size;
  const size_t pe = (size_t)D->plane * s;
  const int64_t bytes = (int64_t)pe * sizeof(double);
  cudaStream_t st = D->ctx->stream;
  struct Msg {
    int from, to;
    cudaEvent_t a, b;
  };
  std::vector<Msg> msgs;
  auto timed = [&](int from, int to, auto&& issue) -> int {
    Msg m{from, to, nullptr, nullptr};
    EP_CUDA(cudaEventCreate(&m.a));
    EP_CUDA(cudaEventCreate(&m.b));
    msgs.push_back(m);
    EP_CUDA(cudaEventRecord(m.a, st));
    int rc = issue();
    if (rc) return rc;
    EP_CUDA(cudaEventRecord(m.b, st));
    return ENPROP_OK;
  };
  int rc = halo(D, 0);  // warm-up (connection setup)
  if (rc) return rc;
  if (D->emulated) {
    for (size_t i = 0; i < D->ranks.size() && !rc; ++i) {
      DistRank& d = D->ranks[i];
      if (i > 0) {
        DistRank& lo = D->ranks[i - 1];
        rc = timed((int)i, (int)i - 1, [&]() -> int {
          EP_CUDA(cudaMemcpyAsync(lo.p[0] + (size_t)(lo.lo_rows + lo.rows) * s, d.p[0] + (size_t)d.lo_rows * s,
                                  pe * sizeof(double), cudaMemcpyDeviceToDevice, st));
          return ENPROP_OK;
        });
      }
      if (!rc && i + 1 < D->ranks.size()) {
        DistRank& hi = D->ranks[i + 1];
        rc = timed((int)i, (int)i + 1, [&]() -> int {
          EP_CUDA(cudaMemcpyAsync(hi.p[0], d.p[0] + (size_t)(d.lo_rows + d.rows - D->plane) * s,
                                  pe * sizeof(double), cudaMemcpyDeviceToDevice, st));
          return ENPROP_OK;
        });
      }
    }
  } else if (D->transport == kIpc) {
    DistRank& d = D->ranks[0];
    rc = ipc_publish(D, kEvP);
    for (int nb : {d.rank - 1, d.rank + 1}) {
      if (rc || nb < 0 || nb >= D->nranks) continue;
      int lo, lr, rws;
      rank_layout(D, nb, lo, lr, rws);
      if ((rc = ipc_wait(D, nb, kEvP))) break;
      rc = timed(nb, d.rank, [&]() -> int {
        double* dst = nb < d.rank ? d.p[0] : d.p[0] + (size_t)(d.lo_rows + d.rows) * s;
        const double* src = D->peer_p[0][nb] + (size_t)(nb < d.rank ? lr + rws - D->plane : lr) * s;
        EP_CUDA(cudaMemcpyAsync(dst, src, pe * sizeof(double), cudaMemcpyDefault, st));
        return ENPROP_OK;
      });
    }
  } else {  // NCCL: each link's send/receive pair as its own group
    DistRank& d = D->ranks[0];
    auto& api = nccl();
    for (int nb : {d.rank - 1, d.rank + 1}) {
      if (rc || nb < 0 || nb >= D->nranks) continue;
      rc = timed(d.rank, nb, [&]() -> int {
        const bool down = nb < d.rank;
        EP_NCCL(api.GroupStart());
        EP_NCCL(api.Send(d.p[0] + (size_t)(down ? d.lo_rows : d.lo_rows + d.rows - D->plane) * s, pe, ncclDouble, nb,
                         D->comm, st));
        EP_NCCL(api.Recv(down ? d.p[0] : d.p[0] + (size_t)(d.lo_rows + d.rows) * s, pe, ncclDouble, nb, D->comm, st));
        EP_NCCL(api.GroupEnd());
        return ENPROP_OK;
      });
    }
  }
  cudaError_t err = cudaStreamSynchronize(st);
  std::vector<double> clock(D->nranks, 0.0);
  double elapsed = 0.0;
  int n = 0;
  for (const Msg& m : msgs) {
    float ms = 0.0f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, m.a, m.b);
    clock[m.from] += ms * 1e-3;
    elapsed = std::max(elapsed, clock[m.from]);
    if (out && n < max_records) out[n] = enprop_exchange_record{m.from, m.to, bytes, clock[m.from]};
    ++n;
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  if (rc) return rc;
  if (err != cudaSuccess) return cuda_fail(err, "enprop_dist_exchange_trace");
  *count = n;
  if (elapsed_seconds) *elapsed_seconds = elapsed;
  return ENPROP_OK;
}

int enprop_fit_halo_model(int n, const double* s, const double* t, double* a, double* b,
                          double* rss) {
  // halo.cpp:156-181, same operations in the same order
  if (n < 2 || !s || !t) return fail(ENPROP_ERR_INVALID, "fit_halo_model: need at least two points");
  double mean_s = 0.0, mean_t = 0.0;
  for (int i = 0; i < n; ++i) {
    mean_s += s[i];
    mean_t += t[i];
  }
  mean_s /= static_cast<double>(n);
  mean_t /= static_cast<double>(n);
  double ss = 0.0, st = 0.0;
  for (int i = 0; i < n; ++i) {
    ss += (s[i] - mean_s) * (s[i] - mean_s);
    st += (s[i] - mean_s) * (t[i] - mean_t);
  }
  if (ss == 0.0) return fail(ENPROP_ERR_INVALID, "fit_halo_model: all ensemble sizes equal, fit is singular");
  const double fb = st / ss;
  const double fa = mean_t - fb * mean_s;
  double r2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = t[i] - fa - fb * s[i];
    r2 += r * r;
  }
  if (a) *a = fa;
  if (b) *b = fb;
  if (rss) *rss = r2;
  return ENPROP_OK;
}

int enprop_predicted_speedup(double a, double b, double s, double* speedup) {
  // halo.cpp:183-188
  if (!speedup) return fail(ENPROP_ERR_INVALID, "predicted_speedup: null output");
  if (s < 1.0) return fail(ENPROP_ERR_INVALID, "predicted_speedup: s must be at least 1");
  const double denom = a + b * s;
  if (denom == 0.0) return fail(ENPROP_ERR_INVALID, "predicted_speedup: zero exchange time");
  *speedup = s * (a + b) / denom;
  return ENPROP_OK;
}

int enprop_dist_stages(enprop_dist* D, int index, int* interior, int* total) {
  if (!D || index < 0 || index >= (int)D->ranks.size()) return fail(ENPROP_ERR_INVALID, "enprop_dist_stages: bad index");
  const DistRank& d = D->ranks[index];
  if (interior) *interior = d.staged ? d.stage.n_interior : 0;
  if (total) *total = d.staged ? d.stage.nstages : 0;
  return ENPROP_OK;
}

int enprop_dist_local_count(enprop_dist* D) { return D ? (int)D->ranks.size() : 0; }

int enprop_dist_local(enprop_dist* D, int index, int* rank, int* row_begin, int* rows, double** x) {
  if (!D || index < 0 || index >= (int)D->ranks.size()) return fail(ENPROP_ERR_INVALID, "enprop_dist_local: bad index");
  const DistRank& d = D->ranks[index];
  if (rank) *rank = d.rank;
  if (row_begin) *row_begin = d.row_begin;
  if (rows) *rows = d.rows;
  if (x) *x = d.x;
  return ENPROP_OK;
}

}  // extern "C"

namespace {

// assemble + Dirichlet of the local ranks' store rows at u (nullptr = 0). With
// u, the caller has put each rank's iterate with its ghost planes into the
// ext-layout p[0] (the u halo, Alg. 2's first step).
int dist_assemble(enprop_dist* D, const double* y, bool with_u) {
  for (auto& d : D->ranks) {
    AsmArgs a = D->setup.args;
    a.rows = d.store_rows;  // staged: the lo ghost plane's upper slots too (no communication)
    a.row_begin = d.row_begin + d.rows - d.store_rows;
    a.kc_lo = d.store_rows > d.rows ? d.k0 - 1 : 0;  // ghost rows: cells toward the owned planes only
    a.u = with_u ? d.p[0] : nullptr;
    a.u_shift = d.ext_begin;
    a.y = y;
    a.row_map = d.row_map;
    a.values = d.values;
    a.residual = d.residual;
    a.vpos = d.vpos;  // full storage (unstaged): nullptr
    a.dirichlet = 1;
    a.bc0 = D->desc.bc.x0_value;
    a.bc1 = D->desc.bc.x1_value;
    EP_CUDA(launch_assemble(D->desc.ensemble_size, a, D->ctx->stream));
    D->ctx->launches += 1;
  }
  return ENPROP_OK;
}

}  // namespace

extern "C" {

int enprop_dist_assemble(enprop_dist* D, const double* y) {
  ScopedLaunchOpts launch_scope(D ? D->ctx : nullptr);
  if (!D || !y) return fail(ENPROP_ERR_INVALID, "enprop_dist_assemble: null argument");
  return dist_assemble(D, y, false);
}

int enprop_dist_solve(enprop_dist* D, const enprop_cg_options* opt, int* iterations, int* lane_status) {
  ScopedLaunchOpts launch_scope(D ? D->ctx : nullptr);
  if (!D || !opt) return fail(ENPROP_ERR_INVALID, "enprop_dist_solve: null argument");
  if (opt->dot_mode != ENPROP_DOT_CANONICAL)
    return fail(ENPROP_ERR_INVALID, "enprop_dist_solve: the multi-GPU solve uses the canonical dot order");
  if (opt->flavour != ENPROP_CG_COUPLED && opt->flavour != ENPROP_CG_UNCOUPLED)
    return fail(ENPROP_ERR_INVALID, "enprop_cg: unknown CG flavour");
  if (opt->max_iterations < 0) return fail(ENPROP_ERR_INVALID, "enprop_cg: negative max_iterations");
  const int s = D->desc.ensemble_size;
  cudaStream_t st = D->ctx->stream;
  enprop_ctx* ctx = D->ctx;
  if (D->maxit < opt->max_iterations) {
    for (auto& d : D->ranks) {
      if (d.hist) cudaFree(d.hist);
      d.hist = nullptr;
      EP_CUDA(cudaMalloc(&d.hist, (size_t)(opt->max_iterations + 1) * s * sizeof(double)));
    }
    D->maxit = opt->max_iterations;
  }
  if (D->transport == kIpc) {  // the init sums reuse the previous solve's RR buffer
    int rc = ipc_quiesce(D);
    if (rc) return rc;
  }
  CgState init;
  std::memset(&init, 0, sizeof(init));
  init.flavour = opt->flavour;
  init.s = s;
  init.maxit = opt->max_iterations;
  init.tol = opt->tol;
  for (auto& d : D->ranks) {
    const size_t vec = (size_t)d.rows * s * sizeof(double);
    EP_CUDA(cudaMemcpyAsync(d.state, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    EP_CUDA(cudaMemsetAsync(d.x, 0, vec, st));
    EP_CUDA(launch_negate((int64_t)d.rows * s, d.residual + (size_t)(d.store_rows - d.rows) * s, d.r,
                          st));  // b = -residual (owned rows); r = b
    EP_CUDA(launch_dot_tiles(s, d.tm, d.r, d.r, rank_fin(d, kPhaseInit), st));
    EP_CUDA(launch_fin_segments(s, d.tm, rank_fin(d, kPhaseInit), st));
    ctx->launches += 3;
  }
  int rc = allgather(D, kPhaseInit);
  if (rc) return rc;
  rc = fin_all(D, kPhaseInit);
  if (rc) return rc;

  const int chunk = opt->check_every > 0 ? opt->check_every : 16;
  const int limit = opt->max_iterations;
  int launched = 0, slot = 0;
  bool pending = false;
  while (true) {
    for (int c2 = 0; c2 < chunk && launched < limit; ++c2, ++launched) {
      const int po = launched & 1, pn = (launched + 1) & 1;
      for (auto& d : D->ranks) {
        EP_CUDA(launch_cg_direction(s, d.rows, d.r, d.p[po] + (size_t)d.lo_rows * s,
                                    d.p[pn] + (size_t)d.lo_rows * s, d.x, d.state, st));
        ctx->launches += 1;
      }
      // halo on the side stream, overlapped with the interior stages (DESIGN.md
      // §7). IPC: the owned planes are published before the interior launch
      // (peers pull them meanwhile), and the pulls are enqueued after it,
      // since waiting for the peers' publishes blocks this host thread.
      EP_CUDA(cudaEventRecord(D->ev_owned, st));
      EP_CUDA(cudaStreamWaitEvent(D->side, D->ev_owned, 0));
      const bool ipc = D->transport == kIpc;
      if ((rc = ipc ? ipc_publish(D, kEvP) : halo(D, pn, D->side))) return rc;
      for (auto& d : D->ranks) {
        if (d.staged && d.stage.n_interior > 0) {  // owned rows only: x runs clipped to [0, rows)
          EP_CUDA(launch_cg_spmv_staged(s, true, false, stage_range(d.stage, 0, d.stage.n_interior, 0, d.rows),
                                        d.values, d.p[pn] + (size_t)d.lo_rows * s, d.q, rank_fin(d, kPhasePQ), st));
          ctx->launches += 1;
        }
      }
      if (ipc && (rc = halo(D, pn, D->side, false))) return rc;
      EP_CUDA(cudaEventRecord(D->ev_halo, D->side));
      EP_CUDA(cudaStreamWaitEvent(st, D->ev_halo, 0));
      for (auto& d : D->ranks) {
        if (d.staged)
          EP_CUDA(launch_cg_spmv_staged(s, true, false,
                                        stage_range(d.stage, d.stage.n_interior, d.stage.nstages - d.stage.n_interior,
                                                    d.stage.xlo, d.stage.xhi),
                                        d.values, d.p[pn] + (size_t)d.lo_rows * s, d.q, rank_fin(d, kPhasePQ), st));
        else
          EP_CUDA(launch_cg_spmv(s, true, false, false, d.tm, d.row_map, d.col_entry, d.values, d.r,
                                 d.p[po] + (size_t)d.lo_rows * s, d.p[pn] + (size_t)d.lo_rows * s, d.q,
                                 d.x, d.p[pn], nullptr, rank_fin(d, kPhasePQ), st));
        EP_CUDA(launch_fin_segments(s, d.tm, rank_fin(d, kPhasePQ), st));
        ctx->launches += 2;
      }
      if ((rc = allgather(D, kPhasePQ)) || (rc = fin_all(D, kPhasePQ))) return rc;
      for (auto& d : D->ranks) {
        EP_CUDA(launch_cg_update(s, true, d.tm, d.r, d.q, rank_fin(d, kPhaseRR), st));
        EP_CUDA(launch_fin_segments(s, d.tm, rank_fin(d, kPhaseRR), st));
        ctx->launches += 2;
      }
      if ((rc = allgather(D, kPhaseRR)) || (rc = fin_all(D, kPhaseRR))) return rc;
    }
    EP_CUDA(cudaMemcpyAsync(&ctx->pinned_flags[slot], &D->ranks[0].state->done, sizeof(int),
                            cudaMemcpyDeviceToHost, st));
    EP_CUDA(cudaEventRecord(ctx->flag_ev[slot], st));
    if (pending) {
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
  for (auto& d : D->ranks) {
    double* pp[2] = {d.p[0] + (size_t)d.lo_rows * s, d.p[1] + (size_t)d.lo_rows * s};
    EP_CUDA(launch_cg_flush(s, d.rows, d.x, pp, d.state, st));
    ctx->launches += 1;
  }
  EP_CUDA(cudaStreamSynchronize(st));
  CgState fin;
  EP_CUDA(cudaMemcpy(&fin, D->ranks[0].state, sizeof(fin), cudaMemcpyDeviceToHost));
  if (!fin.done) return fail(ENPROP_ERR_CUDA, "enprop_dist_solve: solver did not finish (internal)");
  const int lanes = opt->flavour == ENPROP_CG_UNCOUPLED ? s : 1;
  for (int l = 0; l < lanes; ++l) {
    if (iterations) iterations[l] = fin.iters[l];
    if (lane_status) lane_status[l] = opt->flavour == ENPROP_CG_UNCOUPLED ? fin.lane_status[l] : fin.status;
  }
  if (fin.status == ENPROP_ERR_NO_CONVERGENCE)
    return fail(ENPROP_ERR_NO_CONVERGENCE, "pcg_solve: no convergence");
  if (fin.status == ENPROP_ERR_INDEFINITE)
    return fail(ENPROP_ERR_INDEFINITE, "pcg_solve: operator not positive definite (p'Ap <= 0)");
  return ENPROP_OK;
}

// newton_solve (fem.hpp:265-302) over the slabs, with Alg. 2's first step:
// every step imports the neighbours' boundary planes of u (the iterate is
// staged in the ext-layout p[0] and exchanged by the solver's own halo), then
// assembles the local rows at u. The coupled residual norm is the canonical
// dot (per-plane sums all-gathered, summed in global plane order, then over
// the lanes). J du = -f is solved by enprop_dist_solve, and u = 1.0*du + 1.0*u.
// Every rank sees the same norms and takes the same decisions. The result is
// bitwise enprop_problem_newton on one GPU with the canonical dot order.
int enprop_dist_newton(enprop_dist* D, const double* y, const enprop_newton_options* opt,
                       int* newton_iterations, int* total_cg_iterations, double* residual_norms,
                       int* num_norms) {
  ScopedLaunchOpts launch_scope(D ? D->ctx : nullptr);
  if (!D || !y || !opt) return fail(ENPROP_ERR_INVALID, "enprop_dist_newton: null argument");
  if (opt->max_iterations < 0) return fail(ENPROP_ERR_INVALID, "newton_solve: negative max_iterations");
  if (opt->linear.dot_mode != ENPROP_DOT_CANONICAL)
    return fail(ENPROP_ERR_INVALID, "enprop_dist_newton: the multi-GPU solve uses the canonical dot order");
  const int s = D->desc.ensemble_size;
  cudaStream_t st = D->ctx->stream;
  double* scratch = nullptr;  // [0, 2s): the axpby coefficients (1.0); [2s, 3s + 1): the norm's lanes
  EP_CUDA(cudaMalloc(&scratch, (3 * s + 1) * sizeof(double)));
  struct FreeOnExit {
    double* q;
    ~FreeOnExit() { cudaFree(q); }
  } free_scratch{scratch};
  std::vector<double> ones(2 * s, 1.0);
  EP_CUDA(cudaMemcpyAsync(scratch, ones.data(), 2 * s * sizeof(double), cudaMemcpyHostToDevice, st));
  for (auto& d : D->ranks) {
    const size_t vec = (size_t)d.rows * s * sizeof(double);
    if (!d.u) EP_CUDA(cudaMalloc(&d.u, vec));
    EP_CUDA(cudaMemsetAsync(d.u, 0, vec, st));  // result.solution = 0 (fem.hpp:271)
  }
  int steps = 0, cg_total = 0, nn = 0;
  double initial = 0.0;
  auto finish = [&](int code) {
    if (newton_iterations) *newton_iterations = steps;
    if (total_cg_iterations) *total_cg_iterations = cg_total;
    if (num_norms) *num_norms = nn;
    for (auto& d : D->ranks) {  // the iterate is reported in each rank's x
      cudaError_t err = cudaMemcpyAsync(d.x, d.u, (size_t)d.rows * s * sizeof(double), cudaMemcpyDeviceToDevice, st);
      if (err != cudaSuccess) return cuda_fail(err, "enprop_dist_newton");
    }
    cudaError_t err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "enprop_dist_newton");
    return code;
  };
  for (int step = 0;; ++step) {
    // u halo (Alg. 2: import the off-rank entries of u), then assemble at u
    for (auto& d : D->ranks)
      EP_CUDA(cudaMemcpyAsync(d.p[0] + (size_t)d.lo_rows * s, d.u, (size_t)d.rows * s * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
    int rc = halo(D, 0);
    if (rc) return rc;
    if ((rc = dist_assemble(D, y, true))) return rc;
    // norm2(system.residual) (fem.hpp:277): coupled, canonical order
    for (auto& d : D->ranks) {
      const double* res = d.residual + (size_t)(d.store_rows - d.rows) * s;
      EP_CUDA(launch_dot_tiles(s, d.tm, res, res, rank_fin(d, kPhaseNone), st));
      EP_CUDA(launch_fin_segments(s, d.tm, rank_fin(d, kPhaseNone), st));
      D->ctx->launches += 2;
    }
    if ((rc = allgather(D, kPhaseNone))) return rc;
    if ((rc = fin_all(D, kPhaseNone, scratch + 2 * s))) return rc;
    double dot = 0.0;
    EP_CUDA(cudaMemcpyAsync(&dot, scratch + 3 * s, sizeof(double), cudaMemcpyDeviceToHost, st));
    EP_CUDA(cudaStreamSynchronize(st));
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
    const int lanes = opt->linear.flavour == ENPROP_CG_UNCOUPLED ? s : 1;
    std::vector<int> its(lanes, 0), ls(lanes, 0);
    rc = enprop_dist_solve(D, &opt->linear, its.data(), ls.data());
    int mx = 0;
    for (int l = 0; l < lanes; ++l) mx = its[l] > mx ? its[l] : mx;
    cg_total += mx;
    if (rc) {
      steps = step;
      const std::string msg = enprop_last_error();
      finish(ENPROP_OK);
      return fail(rc, msg);
    }
    for (auto& d : D->ranks) {  // axpby(1.0, du, 1.0, u) (fem.hpp:300)
      EP_CUDA(launch_axpby(s, d.rows, 0, scratch, scratch + s, d.x, d.u, st));
      D->ctx->launches += 1;
    }
  }
}

}  // extern "C"
