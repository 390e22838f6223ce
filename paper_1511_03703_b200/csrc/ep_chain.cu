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
//  * warp 1 lane 0 produces: rows arrive as 48 KB stages (per operand) via
//    cp.async.bulk into a 3-stage ring (2 for two operands), completing on
//    mbarriers; the producer alone waits on `empty` barriers, so copy issue
//    stays off the chain;
//  * the consumer walks a stage in fully unrolled 96-row blocks (the compiler
//    hoists the block's shared-memory loads ahead of its DADDs), which runs at
//    the DADD latency; what remains per stage is one `full` wait.
// Measured alternatives (chain_bench.cu): register-prefetched global loads
// (one warp, no shared memory) ran at 25-40 cycles per row (the loads' shared
// scoreboards expose a full L2/HBM latency per batch); small co-resident
// shared-memory rings (<= 16 KB) at 20-80 (too few bytes in flight for the
// ~900-cycle TMA latency, and every consumer-side barrier probe stalls issue);
// register-batched consumption of a big ring at 16-19 (moves + batch waits);
// ring shape (A/B, profiles/round2/README.md §3, 24 groups): 16 KB stages x 4
// / 6 gave 494-503 samples/s, x 8 548-569; 32 KB x 4 (the same 128 KB, half the
// per-stage waits) 574-577, with the p.q / r.r chains at 1.41 / 1.63 ms
// vs 1.57 / 1.84 ms for 16 KB x 8; 48 KB x 3 with 96-row blocks: chains
// 1.32 / 1.60 ms, +0.2-0.4% at 24 groups (same box). A software-pipelined consumer (the next
// 32-row block's terms formed ahead) ran at ~18 cycles per row: ptxas issued
// the next block as one run before the DADDs, plus the register copies.
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

constexpr int kChainChunkBytes = 49152;  // per operand vector per stage
constexpr int kChainBlock = 96;          // rows per unrolled consumer block

template <int NV, int CB = kChainChunkBytes>
struct ChainRing {
  static constexpr int STAGE = CB * NV;
  static constexpr int D = (NV == 1 ? 147456 : 196608) / STAGE;  // stages in the ring (3 x 48 KB / 2 x 96 KB)
  static constexpr int SMEM = D * STAGE + 2 * D * 8;
};

template <int S, int KIND>
__device__ __forceinline__ double chain_term(const double* a, const double* b, int i) {
  const double x = a[i * S];
  if constexpr (KIND == kChainGiven) return x;
  else if constexpr (KIND == kChainSquare) return EP_DMUL(x, x);
  else return EP_DMUL(x, b[i * S]);
}

template <int S, int KIND, int CB>
__global__ void __launch_bounds__(64, 1) k_chain(int rows, const double* __restrict__ u,
                                                 const double* __restrict__ v, const FinArgs f) {
  EP_PDL_ENTRY();
  if ((f.phase == kPhasePQ || f.phase == kPhaseRR) && f.cg->done) return;
  constexpr int NV = KIND == kChainProduct ? 2 : 1;
  using Ring = ChainRing<NV, CB>;
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

bool chain_aligned(const void* u, const void* v) {
  return ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
}

template <int S, int KIND, int CB = kChainChunkBytes>
static cudaError_t chain_sk(int rows, const double* u, const double* v, const FinArgs& f, cudaStream_t st) {
  constexpr int NV = KIND == kChainProduct ? 2 : 1;
  constexpr int SMEM = ChainRing<NV, CB>::SMEM;
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
      err = cudaFuncSetAttribute(k_chain<S, KIND, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
      if (err != cudaSuccess) return err;
      ready[dev].store(1, std::memory_order_release);
    }
  }
  // highest launch priority: a group's latency-critical chain takes the next
  // free SM ahead of other groups' pending SpMV CTAs (+0.3-0.6% at 24 groups)
  launch_kk(4 | kLaunchUrgent, k_chain<S, KIND, CB>, dim3(1), dim3(64), SMEM, st, rows, u, v, f);
  return cudaGetLastError();
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
