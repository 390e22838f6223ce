// Serial (reference-order) dot products for the CG loop and enprop_dot.
//
// The reference's dot (kernels.hpp:62-69) is, per sample e,
//   acc = 0.0;  for row = 0, 1, ...:  acc = acc + u[row][e]*v[row][e]
// followed by reduce_sum over the samples (ensemble.hpp:240-244).  The sum is
// one dependent DADD per row: its latency (8.0 cycles measured,
// tools/microbench/chain_bench.cu) times the row count is a floor no
// reassociation may lower, since every intermediate rounding must be the
// reference's.  The kernel's job is to feed that chain at its own pace:
//
//  * one CTA per dot; warp 0 consumes: lane e < S runs sample e's chain, so a
//    row's S values are one contiguous 8S-byte read from shared memory and the
//    chain never hands off between lanes;
//  * warp 1 lane 0 produces: rows arrive as 32 KB stages (per operand) via
//    cp.async.bulk into a 4-stage ring (3 for two operands), completing on
//    mbarriers; the
//    producer alone waits on `empty` barriers, so copy issue stays off the
//    chain;
//  * the consumer walks a stage in fully unrolled 64-row blocks (the compiler
//    hoists the block's shared-memory loads ahead of its DADDs), which runs at
//    the DADD latency; what remains per stage is one `full` wait.
// Measured alternatives (chain_bench.cu): register-prefetched global loads
// (one warp, no shared memory) ran at 25-40 cycles per row (the loads' shared
// scoreboards expose a full L2/HBM latency per batch); small co-resident
// shared-memory rings (<= 16 KB) at 20-80 (too few bytes in flight for the
// ~900-cycle TMA latency, and every consumer-side barrier probe stalls issue);
// register-batched consumption of a big ring at 16-19 (moves + batch waits).
// The CG scalar phase (ep_fin.cuh cg_phase) runs in the consumer warp.
//
// In the CG loop the SpMV writes the products p*q (f.prod) and the r.r chain
// squares r itself, so each chain reads one vector.
#include <atomic>
#include <mutex>

#include "ep_common.cuh"
#include "ep_fin.cuh"
#include "ep_kernels.h"

namespace ep {

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

constexpr int kChainChunkBytes = 16384;  // per operand vector per stage
constexpr int kChainBlock = 64;          // rows per unrolled consumer block

template <int NV, int D_ = (NV == 1 ? 8 : 6), int CB = kChainChunkBytes>
struct ChainRing {
  static constexpr int STAGE = CB * NV;
  static constexpr int D = D_;  // stages in the ring (default 128 / 192 KB)
  static constexpr int SMEM = D * STAGE + 2 * D * 8;
};

// ENPROP_CHAIN_STAGES (A/B): ring depth of the one-operand chains, 4 or 8
// (default); 4 stages (64 KB) let a chain CTA share an SM with a staged-SpMV
// CTA of the two-per-SM layout
int chain_stages() {
  static const int v = [] {
    const int e = env_int("ENPROP_CHAIN_STAGES", 8);
    return e == 4 || e == 6 || e == 10 || e == 12 ? e : 8;
  }();
  return v;
}

template <int S, int KIND>
__device__ __forceinline__ double chain_term(const double* a, const double* b, int i) {
  const double x = a[i * S];
  if constexpr (KIND == kChainGiven) return x;
  else if constexpr (KIND == kChainSquare) return EP_DMUL(x, x);
  else return EP_DMUL(x, b[i * S]);
}

template <int S, int KIND, int DEPTH, int CB>
__global__ void __launch_bounds__(64, 1) k_chain(int rows, const double* __restrict__ u,
                                                 const double* __restrict__ v, const FinArgs f) {
  EP_PDL_ENTRY();
  if ((f.phase == kPhasePQ || f.phase == kPhaseRR) && f.cg->done) return;
  constexpr int NV = KIND == kChainProduct ? 2 : 1;
  using Ring = ChainRing<NV, DEPTH, CB>;
  constexpr int D = Ring::D;
  constexpr int R = CB / (8 * S);  // rows per stage
  constexpr int BLK = R < kChainBlock ? R : kChainBlock;
  static_assert(R % BLK == 0, "stage must hold whole blocks");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + D * Ring::STAGE);
  uint64_t* empty = full + D;
  __shared__ double lanes[32];
  const int nchunks = (rows + R - 1) / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < D; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 32) {  // ---------------------------------------- producer
    for (int c = 0; c < nchunks; ++c) {
      const int slot = c % D;
      if (c >= D) mbar_wait(&empty[slot], ((c / D) - 1) & 1);
      const int r0 = c * R;
      const int nr = imin(R, rows - r0);
      // bulk sizes are 16-byte multiples: at S = 1 an odd last row is read
      // by the consumer from global memory instead
      const uint32_t bytes = (uint32_t)(S == 1 ? (nr & ~1) : nr) * 8u * S;
      mbar_arrive_expect_tx(&full[slot], bytes * NV);
      if (bytes) {
        bulk_g2s(smem + slot * Ring::STAGE, u + (size_t)r0 * S, bytes, &full[slot]);
        if constexpr (NV == 2)
          bulk_g2s(smem + slot * Ring::STAGE + CB, v + (size_t)r0 * S, bytes, &full[slot]);
      }
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  // -------------------------------------------------------------- consumer
  const int e = threadIdx.x;
  const int el = e < S ? e : 0;  // idle lanes shadow lane 0 (results unused)
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int slot = c % D;
    mbar_wait(&full[slot], (c / D) & 1);
    const double* a = reinterpret_cast<const double*>(smem + slot * Ring::STAGE) + el;
    const double* b = a + CB / 8;
    const int nr = imin(R, rows - c * R);
    if (nr == R) {
      // a block's terms (loads and, for squares / products, the DMULs) are
      // formed before its add chain, so only the DADDs are dependent
#pragma unroll 1
      for (int r0 = 0; r0 < R; r0 += BLK) {
        double t[BLK];
#pragma unroll
        for (int i = 0; i < BLK; ++i) t[i] = chain_term<S, KIND>(a, b, r0 + i);
#pragma unroll
        for (int i = 0; i < BLK; ++i) acc = EP_DADD(acc, t[i]);
      }
    } else {  // last, partial stage
      const int nb = S == 1 ? (nr & ~1) : nr;
      for (int i = 0; i < nb; ++i) acc = EP_DADD(acc, (chain_term<S, KIND>(a, b, i)));
      if (nb < nr) {  // S = 1, odd row count: the last row straight from global memory
        const size_t g = (size_t)(c * R + nr - 1);
        const double x = u[g];
        const double y = KIND == kChainSquare ? x : (KIND == kChainProduct ? v[g] : 1.0);
        const double t = KIND == kChainGiven ? x : EP_DMUL(x, y);
        acc = EP_DADD(acc, t);
      }
    }
    __syncwarp();
    if (e == 0) mbar_arrive(&empty[slot]);
  }
  if (e < S) lanes[e] = acc;
  __syncwarp();
  cg_phase<S>(f.phase, lanes, f.cg, f.hist, f.lanes_out);
}

// Co-resident variant (ENPROP_CHAIN=small): one warp and a 3 x 4 KB ring, so
// the CTA fits beside a persistent staged-SpMV CTA (which leaves ~8 K
// registers and ~17 KB of shared memory per SM) and never keeps one off its
// SM. Lane 0 refills the slot it just consumed and prefetches kSmallAhead rows
// into L2; the chain runs at ~25 cycles per row (chain_bench.cu "tma S32 4KB
// x3 pf1024"), slower than k_chain, which concurrency across sample groups hides.
constexpr int kSmallStage = 4096;
constexpr int kSmallStages = 3;
constexpr int kSmallAhead = 1024;

template <int S, int KIND>
__global__ void __launch_bounds__(32, 1) k_chain_small(int rows, const double* __restrict__ u,
                                                       const double* __restrict__ v, const FinArgs f) {
  EP_PDL_ENTRY();
  if ((f.phase == kPhasePQ || f.phase == kPhaseRR) && f.cg->done) return;
  constexpr int NV = KIND == kChainProduct ? 2 : 1;
  constexpr int SB = kSmallStage / NV;  // bytes per operand per stage
  constexpr int R = SB / (8 * S);       // rows per stage
  constexpr int BLK = R < kChainBlock ? R : kChainBlock;
  constexpr int D = kSmallStages;
  static_assert(R % BLK == 0 && R >= 2, "stage must hold whole blocks");
  __shared__ __align__(128) unsigned char ring[D * kSmallStage];
  __shared__ uint64_t full[D];
  __shared__ double lanes[32];
  const int e = threadIdx.x;
  const int el = e < S ? e : 0;
  const int nchunks = (rows + R - 1) / R;
  if (e == 0) {
    for (int k = 0; k < D; ++k) mbar_init(&full[k], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int c) {  // lane 0: stage c into its slot (+ L2 prefetch ahead)
    if (c >= nchunks) return;
    const int slot = c % D;
    const int r0 = c * R;
    const int nr = imin(R, rows - r0);
    const uint32_t bytes = (uint32_t)(S == 1 ? (nr & ~1) : nr) * 8u * S;
    const int pr = r0 + kSmallAhead;
    if (pr < rows) {
      const uint32_t pb = (uint32_t)imin(R, rows - pr) * 8u * S & ~15u;
      if (pb) {
        prefetch_l2(u + (size_t)pr * S, pb);
        if constexpr (NV == 2) prefetch_l2(v + (size_t)pr * S, pb);
      }
    }
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&full[slot], bytes * NV);
    if (bytes) {
      bulk_g2s(ring + slot * kSmallStage, u + (size_t)r0 * S, bytes, &full[slot]);
      if constexpr (NV == 2) bulk_g2s(ring + slot * kSmallStage + SB, v + (size_t)r0 * S, bytes, &full[slot]);
    }
  };
  if (e == 0) {
    for (int r0 = 0; r0 < kSmallAhead && r0 < rows; r0 += R) {
      const uint32_t pb = (uint32_t)imin(R, rows - r0) * 8u * S & ~15u;
      if (pb) {
        prefetch_l2(u + (size_t)r0 * S, pb);
        if constexpr (NV == 2) prefetch_l2(v + (size_t)r0 * S, pb);
      }
    }
    for (int c = 0; c < D; ++c) issue(c);
  }
  double acc = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int slot = c % D;
    mbar_wait(&full[slot], (c / D) & 1);
    const double* a = reinterpret_cast<const double*>(ring + slot * kSmallStage) + el;
    const double* b = a + SB / 8;
    const int nr = imin(R, rows - c * R);
    if (nr == R) {
#pragma unroll 1
      for (int r0 = 0; r0 < R; r0 += BLK) {
#pragma unroll
        for (int i = 0; i < BLK; ++i) acc = EP_DADD(acc, (chain_term<S, KIND>(a, b, r0 + i)));
      }
    } else {
      const int nb = S == 1 ? (nr & ~1) : nr;
      for (int i = 0; i < nb; ++i) acc = EP_DADD(acc, (chain_term<S, KIND>(a, b, i)));
      if (nb < nr) {
        const size_t g = (size_t)(c * R + nr - 1);
        const double x = u[g];
        const double y = KIND == kChainSquare ? x : (KIND == kChainProduct ? v[g] : 1.0);
        const double t = KIND == kChainGiven ? x : EP_DMUL(x, y);
        acc = EP_DADD(acc, t);
      }
    }
    __syncwarp();
    if (e == 0) issue(c + D);
  }
  if (e < S) lanes[e] = acc;
  __syncwarp();
  cg_phase<S>(f.phase, lanes, f.cg, f.hist, f.lanes_out);
}

// ENPROP_CHAIN (A/B): 0 = k_chain (default), 1 = k_chain_small
int chain_mode() {
  static const int m = env_int("ENPROP_CHAIN", 0);
  return m;
}

bool chain_aligned(const void* u, const void* v) {
  return ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
}

template <int S, int KIND, int DEPTH, int CB = kChainChunkBytes>
static cudaError_t chain_skd(int rows, const double* u, const double* v, const FinArgs& f, cudaStream_t st) {
  constexpr int NV = KIND == kChainProduct ? 2 : 1;
  constexpr int SMEM = ChainRing<NV, DEPTH, CB>::SMEM;
  // shared-memory opt-in once per device (solves on several host threads)
  static std::atomic<int> ready[64];
  static std::mutex mu;
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!ready[dev].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(mu);
    if (!ready[dev].load(std::memory_order_relaxed)) {
      err = cudaFuncSetAttribute(k_chain<S, KIND, DEPTH, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
      if (err != cudaSuccess) return err;
      ready[dev].store(1, std::memory_order_release);
    }
  }
  if (chain_mode() == 1) launch_kk(4, k_chain_small<S, KIND>, dim3(1), dim3(32), 0, st, rows, u, v, f);
  else launch_kk(4, k_chain<S, KIND, DEPTH, CB>, dim3(1), dim3(64), SMEM, st, rows, u, v, f);
  return cudaGetLastError();
}

// ENPROP_CHAIN_CHUNK (A/B): bytes per operand per stage, 32768 (default: 4
// stages, 128 KB) or 16384 (8 stages, the same ring bytes). The larger stage
// halves the per-stage barrier waits: 64^3, s = 32, p.q 1.57 -> 1.41 ms,
// r.r 1.85 -> 1.66 ms per dot (tools/serial_ab.py)
int chain_chunk() {
  static const int v = env_int("ENPROP_CHAIN_CHUNK", 32768) == 16384 ? 16384 : 32768;
  return v;
}

template <int S, int KIND>
static cudaError_t chain_sk(int rows, const double* u, const double* v, const FinArgs& f, cudaStream_t st) {
  if (chain_chunk() == 32768 && chain_stages() == 8)
    return chain_skd<S, KIND, KIND == kChainProduct ? 3 : 4, 32768>(rows, u, v, f, st);
  if (KIND != kChainProduct && chain_stages() == 4) return chain_skd<S, KIND, 4>(rows, u, v, f, st);
  if (KIND != kChainProduct && chain_stages() == 6) return chain_skd<S, KIND, 6>(rows, u, v, f, st);
  if (KIND != kChainProduct && chain_stages() == 10) return chain_skd<S, KIND, 10>(rows, u, v, f, st);
  if (KIND != kChainProduct && chain_stages() == 12) return chain_skd<S, KIND, 12>(rows, u, v, f, st);
  return chain_skd<S, KIND, KIND == kChainProduct ? 6 : 8>(rows, u, v, f, st);
}

template <int S>
static cudaError_t chain_s(int rows, const double* u, const double* v, int kind, const FinArgs& f,
                           cudaStream_t st) {
  if (kind == kChainGiven) return chain_sk<S, kChainGiven>(rows, u, v, f, st);
  if (kind == kChainSquare) return chain_sk<S, kChainSquare>(rows, u, v, f, st);
  return chain_sk<S, kChainProduct>(rows, u, v, f, st);
}

cudaError_t launch_chain(int s, int rows, const double* u, const double* v, int kind, const FinArgs& f,
                         cudaStream_t st) {
  EP_DISPATCH_S(s, chain_s, rows, u, v, kind, f, st);
}

}  // namespace ep
