// Stage-pipelined CG SpMV for structured-mesh problems with symmetric storage
// ("staged SpMV").
//
// Same arithmetic as k_cg_spmv_warp (ep_kernels.cu): row sums in column order,
// z = ((0 + a_0 x_0) + a_1 x_1) + ... per sample (kernels.hpp:15-26), and the
// same canonical 16-row tile trees for p.q, so the two kernels are bitwise
// interchangeable.  What changes is how the bytes reach the SM.
//
// A stage is T = 32/S consecutive canonical tiles (16 T rows, a contiguous row
// range [R0, R1)).  One persistent CTA per SM walks the stages in a band sweep
// order (CTA c takes sweep positions c, c + grid, ...; a band of mesh lines is
// swept through all planes before the next band, so the upper slots a row
// reads transposed are still in L2) through a two-deep ring of shared-memory
// stage buffers.  Thread 0 fills a buffer with cp.async.bulk (TMA engine)
// copies completing on an mbarrier:
//   * the stage's stored slots (diagonal + upper of its rows): one contiguous
//     range of the symmetric value array, up to 16 T x 14 x 8S = 57 KB;
//   * the direction vector around the stage: the 27-point neighbours of rows
//     [R0, R1) lie in 9 contiguous row runs [R0-1 + dj N + dk N^2, R1+1 + ...),
//     dj, dk in {-1,0,1} (x-fastest numbering, mesh.hpp:24-26), 9 x 18 x 8S
//     bytes at S = 32 instead of 16 x 27 gathers;
//   * a precomputed index block (k_stage_fill, its own ring): per row slot
//     the row and local row, per stencil slot (27, column order) where the
//     value lives; x of slot (run, di) is at position lr + di + 1 of x run
//     `run` (computed).
// Only the lower entries whose transposed slot belongs to an earlier stage
// (<= 13 per row, the leading stencil slots) are gathered from global memory
// into registers, one stage ahead.  The register file therefore only holds
// the transposed gathers; the streamed bytes are in flight in the TMA engine.
// With tiles, the kernel also closes the p.q dot: after a grid barrier
// (cooperative launch) the CTAs fold the canonical segments and the last one
// runs the CG phase (ep_fin.cuh), replacing the separate finalize launch.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ep_common.cuh"
#include "ep_kernels.h"
#include "ep_fin.cuh"

namespace ep {

// NB = stage buffers per CTA: 2 (one persistent CTA per SM, the next stage's
// buffer and transposed gathers in flight during the current one) or 1 (two
// CTAs per SM at <= 128 registers: each CTA loads one stage while the other
// computes; ENPROP_STAGED_CTAS=2).
template <int S, int NB = 2>
struct StagedShape {
  static constexpr int V = 2;
  static constexpr int TPR = S / V;                 // threads per row
  static constexpr int T = 32 / S;                  // canonical tiles per stage
  static constexpr int RS = kTileRows * T;          // row slots per stage
  static constexpr int L = RS + 2;                  // rows per x run
  static constexpr int CH = 8 * S;                  // bytes per chunk (one entry's / row's s values)
  static constexpr int ROWE = 28;                   // value codes per row slot: 27 stencil slots + pad
  static constexpr int UP_CHUNKS = RS * kStageMaxUpper;
  static constexpr int X_CHUNKS = 9 * L;
  static constexpr int ZC = UP_CHUNKS + X_CHUNKS;   // the zero chunk (padding entries)
  static constexpr int BIG_BYTES = ((ZC + 1) * CH + 127) / 128 * 128;
  static constexpr int HDR = 2 * RS + 4;            // ints: srow[RS], slr[RS], stage id, pad
  static constexpr int IDX_BYTES = HDR * 4 + RS * ROWE * 4;
  static constexpr int NIDX = (S >= 16 && NB == 2) ? 4 : 2;  // index blocks in flight (ring depth; smem-limited)
  static constexpr int RED_BYTES = RS * S * 8;
  static constexpr int PFMAX = 3;                    // L2 prefetch distance beyond the stage buffers (max)
  static constexpr int CLAIM = NB + PFMAX + 1 > NIDX ? NB + PFMAX + 1 : NIDX;  // stages claimed ahead
  static constexpr int SMEM = NB * BIG_BYTES + NIDX * IDX_BYTES + 2 * RED_BYTES + 64 + 32;
  static_assert(RS * TPR == 256, "one thread per (row slot, sample pair)");
  static_assert(BIG_BYTES % 128 == 0 && IDX_BYTES % 16 == 0, "alignment");
  static_assert(SMEM <= (NB == 2 ? 232448 : 115712), "stage ring exceeds shared memory");
  static_assert(ZC < 65536, "chunk indices are 16-bit");
};

// the transposed gathers of one stage (the first kStageMaxGlobal entries of a
// row may live in an earlier stage) and the codes of entries 0..15
struct StageGather {
  int code[16];
  double2 v[kStageMaxGlobal];
};

template <int S, int NB = 2>
struct StagedCta {
  using Sh = StagedShape<S, NB>;
  const TileMap& tm;
  int N, nstages, xlo, xhi;
  const StageDesc* __restrict__ desc;
  const unsigned char* __restrict__ blk;
  const double* __restrict__ values;
  const double* __restrict__ p;
  double* __restrict__ q;
  const FinArgs& f;
  unsigned char* smem;
  uint64_t* bar;  // [0,NB): big buffers, [NB,NB+NIDX): index ring
  double* red;
  int* claims;    // [8] sweep positions of this CTA's stages it, it+1, ... (ring)
  int* ticket;    // global claim counter (f.ticket)
  uint64_t pol;
  int rr, lane0;
  int pf;                      // ENPROP_STAGED_PF: L2 prefetch distance in stages beyond the buffers

  // The it-th stage of this CTA is the sweep position it claimed it-th (desc
  // and index blocks are stored in sweep order; desc[pos].g is the stage's
  // canonical id). Claims are dynamic: thread 0 draws tickets from a global
  // counter CLAIM stages ahead, so the positions in flight across all CTAs
  // stay a contiguous window of the sweep whatever the CTAs' start times (a
  // CTA that starts late, e.g. behind another group's kernel on its SM, simply
  // gets fewer stages). Every CTA draws exactly one ticket >= nstages; the
  // CTA that draws the last of them (nstages + grid - 1) resets the counter.
  __device__ __forceinline__ int stage_of(int it) const { return claims[it & 7]; }
  __device__ __forceinline__ bool has(int it) const { return stage_of(it) < nstages; }
  // thread 0 only; claims must be made in order it = 0, 1, ...
  __device__ __forceinline__ void claim(int it) const {
    if (it > 0 && !has(it - 1)) {
      claims[it & 7] = nstages;
      return;
    }
    const int t = atomicAdd(ticket, 1);
    if (t == nstages + (int)gridDim.x - 1) *ticket = 0;
    claims[it & 7] = t < nstages ? t : nstages;
  }
  __device__ __forceinline__ unsigned char* big(int it) const { return smem + (it & (NB - 1)) * Sh::BIG_BYTES; }
  __device__ __forceinline__ uint64_t* big_bar(int it) const { return &bar[it & (NB - 1)]; }
  __device__ __forceinline__ uint32_t big_parity(int it) const { return (it / NB) & 1; }
  __device__ __forceinline__ uint64_t* idx_bar(int it) const { return &bar[NB + (it & (Sh::NIDX - 1))]; }
  __device__ __forceinline__ const int* idx(int it) const {
    return reinterpret_cast<const int*>(smem + NB * Sh::BIG_BYTES + (it & (Sh::NIDX - 1)) * Sh::IDX_BYTES);
  }

  // producer (thread 0)
  __device__ __forceinline__ void issue_big(int it, const StageDesc& d) const {
    unsigned char* sb = big(it);
    uint64_t* b = big_bar(it);
    const int NN = N * N;
    const int L = d.R1 - d.R0 + 2;
    const uint32_t upb = (uint32_t)(d.slot1 - d.slot0) * Sh::CH;
    uint32_t total = upb;
#pragma unroll
    for (int run = 0; run < 9; ++run) {
      const int a = d.R0 - 1 + (run % 3 - 1) * N + (run / 3 - 1) * NN;
      const int lo = a > xlo ? a : xlo, hi = a + L < xhi ? a + L : xhi;
      if (hi > lo) total += (uint32_t)(hi - lo) * Sh::CH;
    }
    mbar_arrive_expect_tx(b, total);
    bulk_g2s(sb, values + (size_t)d.slot0 * S, upb, b);
#pragma unroll
    for (int run = 0; run < 9; ++run) {
      const int a = d.R0 - 1 + (run % 3 - 1) * N + (run / 3 - 1) * NN;
      const int lo = a > xlo ? a : xlo, hi = a + L < xhi ? a + L : xhi;
      if (hi > lo)
        bulk_g2s(sb + (size_t)(Sh::UP_CHUNKS + run * Sh::L + (lo - a)) * Sh::CH, p + (ptrdiff_t)lo * S,
                 (uint32_t)(hi - lo) * Sh::CH, b);
    }
  }
  // L2 prefetch of a later stage's HBM-fresh bytes: its stored slots and the
  // x runs of the plane ahead (dk = +1; the other runs were read by earlier stages)
  __device__ __forceinline__ void prefetch_stage(const StageDesc& d) const {
    const uint32_t upb = (uint32_t)(d.slot1 - d.slot0) * Sh::CH;
    if (upb) prefetch_l2_bulk(values + (size_t)d.slot0 * S, upb);
    const int NN = N * N, L = d.R1 - d.R0 + 2;
#pragma unroll
    for (int run = 6; run < 9; ++run) {
      const int a = d.R0 - 1 + (run % 3 - 1) * N + NN;
      const int lo = a > xlo ? a : xlo, hi = a + L < xhi ? a + L : xhi;
      if (hi > lo) prefetch_l2_bulk(p + (ptrdiff_t)lo * S, (uint32_t)(hi - lo) * Sh::CH);
    }
  }
  __device__ __forceinline__ void issue_idx(int it) const {
    uint64_t* b = idx_bar(it);
    mbar_arrive_expect_tx(b, Sh::IDX_BYTES);
    bulk_g2s((void*)idx(it), blk + (size_t)stage_of(it) * Sh::IDX_BYTES, Sh::IDX_BYTES, b);
  }

  __device__ __forceinline__ void gather(int it, StageGather& G) const {
    const int4* sa = reinterpret_cast<const int4*>(idx(it) + Sh::HDR + rr * Sh::ROWE);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int4 w = sa[v];
      G.code[4 * v] = w.x, G.code[4 * v + 1] = w.y, G.code[4 * v + 2] = w.z, G.code[4 * v + 3] = w.w;
    }
#pragma unroll
    for (int k = 0; k < kStageMaxGlobal; ++k) {
      if (G.code[k] >= 0) {
        const VecD<2> v = ld_stream_hint<2>(values + (size_t)G.code[k] * S + lane0, pol);
        G.v[k] = make_double2(v.v[0], v.v[1]);
      }
    }
  }

  // in-stage value code: 0x80000000 | (byte offset >> 4); (code << 4) drops the flag
  __device__ __forceinline__ double2 slot_val(const unsigned char* lb, int c) const {
    return *reinterpret_cast<const double2*>(lb + ((uint32_t)c << 4));
  }
  __device__ __forceinline__ double2 chunk(const unsigned char* sb, int c) const {
    return *reinterpret_cast<const double2*>(sb + c * Sh::CH + lane0 * 8);
  }

  // NB = 2: Gc holds this stage's gathers (issued one stage ahead), Gn
  // receives the next stage's; NB = 1: Gc is gathered here (Gn unused)
  template <bool kTiles>
  __device__ __forceinline__ void stage(int it, StageGather& Gc, StageGather& Gn) const {
    StageDesc dn, dp;  // producer: descriptors of stage it + NB (and it + NB + pf), loaded early
    const bool prod = threadIdx.x == 0 && has(it + NB);
    if (prod) dn = desc[stage_of(it + NB)];
    const bool pfetch = threadIdx.x == 0 && pf > 0 && has(it + NB + pf);
    if (pfetch) dp = desc[stage_of(it + NB + pf)];
    if constexpr (NB == 2) {
      if (has(it + 1)) {  // the next stage's transposed gathers fly during this stage
        mbar_wait(idx_bar(it + 1), ((it + 1) / Sh::NIDX) & 1);
        gather(it + 1, Gn);
      }
    } else {
      mbar_wait(idx_bar(it), (it / Sh::NIDX) & 1);
      gather(it, Gc);
    }
    const int* ib = idx(it);
    const int row = ib[rr];
    const int lr = ib[Sh::RS + rr];  // local row (x-run positions)
    int ca[12];  // codes of stencil slots 16..27
    {
      const int4* sa = reinterpret_cast<const int4*>(ib + Sh::HDR + rr * Sh::ROWE) + 4;
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const int4 w = sa[v];
        ca[4 * v] = w.x, ca[4 * v + 1] = w.y, ca[4 * v + 2] = w.z, ca[4 * v + 3] = w.w;
      }
    }
    mbar_wait(big_bar(it), big_parity(it));
    const unsigned char* sb = big(it);
    // Stencil slots k = run*3 + di + 1 in column order, run = (dk+1)*3 + dj+1;
    // absent neighbours (and empty row slots) point the value at the zero chunk
    // and add +0.0 * x (the running sum starts at +0.0 and never becomes
    // -0.0, so adding a signed zero changes no bit).  x of slot (run, di) sits
    // at position lr + di + 1 of x run `run`.
    double s0 = 0.0, s1 = 0.0;
    double2 pown = make_double2(0.0, 0.0);
    const unsigned char* lb = sb + lane0 * 8;  // this thread's samples in chunk 0
    const unsigned char* xb = lb + Sh::UP_CHUNKS * Sh::CH + lr * Sh::CH;
#pragma unroll
    for (int run = 0; run < 9; ++run) {
      const unsigned char* xr = xb + run * Sh::L * Sh::CH;
      const double2 xm = *reinterpret_cast<const double2*>(xr);
      const double2 x0 = *reinterpret_cast<const double2*>(xr + Sh::CH);
      const double2 xp = *reinterpret_cast<const double2*>(xr + 2 * Sh::CH);
      if (run == 4) pown = x0;  // the row's own p
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int k = run * 3 + d;
        const int c = k < 16 ? Gc.code[k] : ca[k - 16];
        double2 a;
        if (k < kStageMaxGlobal) {
          a = Gc.v[k];
          if (c < 0) a = slot_val(lb, c);
        } else {
          a = slot_val(lb, c);
        }
        const double2 xv = d == 0 ? xm : (d == 1 ? x0 : xp);
        s0 = EP_DADD(s0, EP_DMUL(a.x, xv.x));
        s1 = EP_DADD(s1, EP_DMUL(a.y, xv.y));
      }
    }
    if (row >= 0) *reinterpret_cast<double2*>(q + (size_t)row * S + lane0) = make_double2(s0, s1);
    if (!kTiles && f.prod && row >= 0)  // serial order: p*q for the chain (kernels.hpp:67)
      *reinterpret_cast<double2*>(f.prod + (size_t)row * S + lane0) =
          make_double2(EP_DMUL(pown.x, s0), EP_DMUL(pown.y, s1));
    double* rb = red + (it & 1) * (Sh::RS * S);
    if constexpr (kTiles) {
      double c0 = 0.0, c1 = 0.0;
      if (row >= 0) {  // own p (x run (dj, dk) = (0, 0))
        c0 = EP_DMUL(pown.x, s0);
        c1 = EP_DMUL(pown.y, s1);
      }
      *reinterpret_cast<double2*>(rb + rr * S + lane0) = make_double2(c0, c1);
    }
    // tile existence (first row slot of each tile), read before the barrier:
    // thread 0 refills this index slot right after it
    // the stage's tile trees run in one warp, rotating over the CTA's warps
    // stage by stage so no warp is late to every barrier
    const int tree_warp = it & 7;
    const int tl = threadIdx.x & 31;
    const bool tree = (threadIdx.x >> 5) == tree_warp;
    const bool tile_exists = tree && ib[(tl / S) * kTileRows] >= 0;
    const int gid = ib[2 * Sh::RS];  // canonical stage id (tile trees)
    __syncthreads();  // big buffer and index slot of stage it consumed, products in rb
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      if (prod) issue_big(it + NB, dn);
      if (pfetch) prefetch_stage(dp);
      claim(it + Sh::CLAIM);
      if (has(it + Sh::NIDX)) issue_idx(it + Sh::NIDX);
    }
    if constexpr (kTiles) {
      if (tree) {  // tile trees: lane -> (tile, sample); v[i] += v[i+h], h = 8,4,2,1
        const int tt = tl / S, e = tl % S;
        const int b2 = gid * Sh::T + tt;
        if (tile_exists) {
          double v[kTileRows];
#pragma unroll
          for (int h = 0; h < kTileRows; ++h) v[h] = rb[(tt * kTileRows + h) * S + e];
#pragma unroll
          for (int h = kTileRows / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int k = 0; k < h; ++k) v[k] = EP_DADD(v[k], v[k + h]);
          f.partials[(size_t)b2 * S + e] = v[0];
        }
      }
    }
  }
};

// Grid-wide barrier of the persistent staged kernel: its grid is one CTA per
// SM (at most), so all CTAs are resident or become resident as other streams'
// kernels retire. Self-resetting counter + monotonic generation.
__device__ __forceinline__ void grid_barrier(int* count, int* gen, int nblocks) {
  // count returns to 0 at every release; gen only grows (its own word: no other
  // counter of the workspace aliases it)
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile int* vgen = gen;
    const int g = *vgen;
    __threadfence();
    if (atomicAdd(count, 1) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1);
    } else {
      while (*vgen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int S, bool kTiles, int NB>
__global__ void __launch_bounds__(256, NB == 2 ? 1 : 2) k_cg_spmv_staged(
    const TileMap tm, int N, int nstages, int xlo, int xhi, const StageDesc* __restrict__ desc,
    const unsigned char* __restrict__ blk, const double* __restrict__ values,
    const double* __restrict__ p, double* __restrict__ q, const FinArgs f, int fuse_fin, int pf) {
  using Sh = StagedShape<S, NB>;
  EP_PDL_ENTRY();
  if (f.cg->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  unsigned char* tail = smem + NB * Sh::BIG_BYTES + Sh::NIDX * Sh::IDX_BYTES + 2 * Sh::RED_BYTES;
  StagedCta<S, NB> c{tm, N, nstages, xlo, xhi, desc, blk, values, p, q, f, smem,
                 reinterpret_cast<uint64_t*>(tail),
                 reinterpret_cast<double*>(smem + NB * Sh::BIG_BYTES + Sh::NIDX * Sh::IDX_BYTES),
                 reinterpret_cast<int*>(tail + 64), f.ticket,
                 l2_policy_evict_normal(), tid / Sh::TPR, (tid % Sh::TPR) * Sh::V, pf};
  if (tid == 0) {
    for (int k = 0; k < NB + Sh::NIDX; ++k) mbar_init(&c.bar[k], 1);
    fence_mbar_init();
    for (int it = 0; it < Sh::CLAIM; ++it) c.claim(it);
  }
  // zero chunks (never written by the copies) and x-run areas: positions a
  // copy does not reach (clipped runs) are read for absent neighbours only,
  // times a zero value, so they must hold finite numbers
  for (int b = 0; b < NB; ++b) {
    double2* z = reinterpret_cast<double2*>(smem + b * Sh::BIG_BYTES + Sh::UP_CHUNKS * Sh::CH);
    for (int i = tid; i < (Sh::X_CHUNKS + 1) * Sh::CH / 16; i += blockDim.x) z[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (tid == 0) {
    fence_proxy_async_smem();  // the zero-filled x areas are rewritten by the copies
    for (int it = 0; it < Sh::NIDX; ++it)
      if (c.has(it)) c.issue_idx(it);
    for (int it = 0; it < NB; ++it)
      if (c.has(it)) c.issue_big(it, desc[c.stage_of(it)]);
    for (int it = NB; it < NB + pf; ++it)
      if (c.has(it)) c.prefetch_stage(desc[c.stage_of(it)]);
  }
  if (c.has(0)) {  // (a CTA may draw no stage at all; it still joins the barrier)
    if constexpr (NB == 2) {
      StageGather ga, gb;
      mbar_wait(c.idx_bar(0), 0);
      c.gather(0, ga);
      for (int it = 0;;) {
        c.template stage<kTiles>(it, ga, gb);
        if (!c.has(++it)) break;
        c.template stage<kTiles>(it, gb, ga);
        if (!c.has(++it)) break;
      }
    } else {
      StageGather g;
      for (int it = 0; c.has(it); ++it) c.template stage<kTiles>(it, g, g);
    }
  }
  if constexpr (kTiles) {
    if (fuse_fin) {
      // Fused canonical finalize (the k_fin_segments work, same order): once
      // every tile partial is written, CTA c folds segments c, c + grid, ...
      // and the last CTA to finish its folds forms the total and runs the CG
      // phase. The stage buffers are free now and serve as scratch.
      grid_barrier(f.bar, f.bar + 1, gridDim.x);
      double* scratch = reinterpret_cast<double*>(smem);
      double* lanes = scratch + FinShape<S>::CHUNK * S + FinShape<S>::CHUNK2 * S;
      int* s_final = reinterpret_cast<int*>(lanes + S);
      int folds = 0;
      for (int seg = blockIdx.x; seg < tm.num_segs; seg += gridDim.x, ++folds)
        fin_segment_fold<S>(tm, f, seg, scratch);
      if (folds) fin_total_phase<S>(tm, f, scratch + FinShape<S>::CHUNK * S, lanes, s_final, folds);
    }
  }
}

// ---- stage map ---------------------------------------------------------------
// Index block of the stage at sweep position pos (blk + pos * IDX_BYTES; the
// stage's canonical id g = desc[pos].g), by row slot rr = ti*16 + t (tile ti
// of the stage, row t of the tile):
//   int srow[RS]       the slot's row, -1 if none
//   int slr[RS]        its local row lr = row - R0 (x-run positions lr .. lr+2);
//                      empty slots: rr for s = 32 (the warp's row pair stays
//                      consecutive), 0 otherwise
//   int g, pad[3]      canonical stage id (tiles g*T + ti)
//   int sa[RS][28]     value of stencil slot k = run*3 + di + 1, run =
//                      (dk+1)*3 + dj+1 (column order): >= 0 global slot (the
//                      transposed entry of an earlier stage's row), else
//                      0x80000000 | (byte offset in the stage buffer >> 4);
//                      absent neighbours and empty slots point at the zero chunk
__global__ void k_stage_fill(const TileMap tm, int nstages, int T, int N, int L, int RS, int ch,
                             int up_chunks, int zc, int idx_bytes,
                             const StageDesc* __restrict__ desc, const int* __restrict__ row_map,
                             const int* __restrict__ col_entry, const int* __restrict__ vpos,
                             unsigned char* __restrict__ blk, int* __restrict__ bad) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nstages * RS) return;
  const int pos = gid / RS, rr = gid % RS;  // sweep position, row slot
  const StageDesc d = desc[pos];
  const int g = d.g;                          // canonical stage id
  int* ib = reinterpret_cast<int*>(blk + (size_t)pos * idx_bytes);
  const int hdr = 2 * RS + 4;
  int* sa = ib + hdr + rr * 28;
  if (rr == 0) ib[2 * RS] = g;  // stage id for the tile trees
  auto smem_code = [&](int chunk) { return (int)(0x80000000u | (uint32_t)(chunk * ch >> 4)); };
  for (int k = 0; k < 28; ++k) sa[k] = smem_code(zc);
  const int b = g * T + rr / kTileRows, t = rr % kTileRows;
  int r0 = 0, nr = 0;
  if (b < tm.num_tiles()) tm.tile(b, r0, nr);
  const int r = t < nr ? r0 + t : -1;
  if (r < 0) {
    ib[rr] = -1;
    ib[RS + rr] = T == 1 ? rr : 0;
    return;
  }
  const int ks = row_map[r], ke = row_map[r + 1];
  const int lr = r - d.R0;
  if (ke - ks > kStageMaxRow || lr < 0 || lr >= RS || (T == 1 && lr != rr)) {
    atomicAdd(bad, 1);
    return;
  }
  const int NN = N * N;
  int last = -1;
  for (int k = ks; k < ke; ++k) {
    const int c = col_entry[k], v = vpos[k];
    const int dl = c - r;
    const int dk = dl > NN / 2 ? 1 : (dl < -(NN / 2) ? -1 : 0);
    const int rem = dl - dk * NN;
    const int dj = rem > N / 2 ? 1 : (rem < -(N / 2) ? -1 : 0);
    const int di = rem - dj * N;
    const int slot = ((dk + 1) * 3 + (dj + 1)) * 3 + di + 1;
    if (di < -1 || di > 1 || slot <= last) atomicAdd(bad, 1);  // 27-point, column order
    last = slot;
    int code;
    if (c >= d.R0) {
      const int a = v - d.slot0;
      if (a < 0 || a >= up_chunks) atomicAdd(bad, 1);
      code = smem_code(a);
    } else {
      if (slot >= kStageMaxGlobal) atomicAdd(bad, 1);
      code = v;
    }
    if (slot >= 0 && slot < 27) sa[slot] = code;
  }
  ib[rr] = r;
  ib[RS + rr] = lr;
}

template <int S>
static int stage_shape(int& T, int& L, int& RS, int& max_upper, int& idx_bytes, int& zc) {
  using Sh = StagedShape<S>;
  T = Sh::T;
  L = Sh::L;
  RS = Sh::RS;
  max_upper = Sh::UP_CHUNKS;
  idx_bytes = Sh::IDX_BYTES;
  zc = Sh::ZC;
  return 0;
}


bool staged_fuse_fin() {
  static const int on = env_int("ENPROP_STAGED_FUSE", 1);
  return on != 0;
}

// ENPROP_STAGED_PF (A/B): L2 prefetch distance in stages beyond the stage
// buffers, 0-3; default 1. The kernel is latency-bound on its stage stream
// (ncu: L1/shared data path 52% busy, issue 7%, stalls on long scoreboard and
// barriers), and a TMA L2 prefetch of the next-but-one stage's HBM-fresh bytes
// (stored slots + the x runs of the plane ahead) makes its shared-memory fill
// an L2 hit: 64^3 s=32 serial-order SpMV 0.249 -> 0.220 ms, 24-group bench
// +4%; 2 stages 0.233, 3 stages 0.316 ms (L2 thrash)
int staged_pf() {
  static const int v = [] {
    const int e = env_int("ENPROP_STAGED_PF", 1);
    return e < 0 ? 0 : (e > 3 ? 3 : e);
  }();
  return v;
}

bool plain_cg_spmv() {
  static const int on = env_int("ENPROP_PLAIN_CG_SPMV", 1);
  return on != 0;
}

// ENPROP_STAGED_SERIAL (A/B, default 1): the staged kernel also serves the
// serial dot order (writing the p*q products); 0 keeps the warp kernel there
bool staged_serial() {
  static const int on = env_int("ENPROP_STAGED_SERIAL", 1);
  return on != 0;
}

// s = 8 measured slower than the warp-per-tile kernel (0.125 vs 0.096 ms at
// 64^3), s = 4 faster (0.081 vs 0.087), s = 16 / 32 faster (tools/kernel_bench.py --ab)
bool staged_supported(int s, int N) { return (s == 4 || s == 16 || s == 32) && N >= 8; }

cudaError_t build_stage_map(int s, const TileMap& tm, int N, const int* row_map,
                            const int* col_entry, const int* vpos, const int* up_start,
                            StageMap& sm, cudaStream_t st, int xlo, int xhi, int interior_lo,
                            int interior_hi) {
  free_stage_map(sm);
  if (!staged_supported(s, N) || tm.rows <= 0 || tm.rows % (N * N) != 0) return cudaErrorInvalidValue;
  int T = 0, L = 0, RS = 0, max_upper = 0, idx_bytes = 0, zc = 0;
  if (s == 32) stage_shape<32>(T, L, RS, max_upper, idx_bytes, zc);
  else if (s == 16) stage_shape<16>(T, L, RS, max_upper, idx_bytes, zc);
  else stage_shape<4>(T, L, RS, max_upper, idx_bytes, zc);
  const int rows = tm.rows;
  std::vector<int> hup(rows + 1);
  cudaError_t err = cudaMemcpyAsync(hup.data(), up_start, (rows + 1) * sizeof(int), cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  if (err != cudaSuccess) return err;
  const int tiles = tm.num_tiles();
  std::vector<StageDesc> hd;
  hd.reserve((tiles + T - 1) / T);
  int64_t off = 0;
  for (int b0 = 0; b0 < tiles; b0 += T) {
    int R0 = -1, R1 = -1;
    for (int ti = 0; ti < T && b0 + ti < tiles; ++ti) {
      int r0, nr;
      tm.tile(b0 + ti, r0, nr);
      if (nr > 0) {
        if (R0 < 0) R0 = r0;
        else if (r0 != R1) return cudaErrorInvalidValue;  // stages must be contiguous
        R1 = r0 + nr;
      }
    }
    if (R0 < 0) break;  // only trailing tiles of the last segment are empty
    StageDesc d{};
    d.R0 = R0;
    d.R1 = R1;
    d.slot0 = hup[R0];
    d.slot1 = hup[R1];
    if (d.slot1 - d.slot0 > max_upper) return cudaErrorInvalidValue;
    d.blk_off = off;
    d.blk_bytes = idx_bytes;
    off += idx_bytes;
    hd.push_back(d);
  }
  sm.nstages = (int)hd.size();
  // Sweep order: stages grouped by bands of B mesh lines (B*N ~ 4096 rows per
  // plane), each band swept through all planes. A row's transposed (lower)
  // slots live one plane back in the same band, ~4096 rows of stored slots
  // (~15 MB at s = 32) earlier in the sweep: still in L2 even when a whole
  // plane is not (256^3: 237 MB of stored slots per plane).
  std::vector<int> ord(hd.size());
  {
    const int NN = N * N;
    const int B = 4096 / N > 1 ? 4096 / N : 1;
    std::vector<int64_t> key(hd.size());
    for (size_t g = 0; g < hd.size(); ++g) {
      const int r = hd[g].R0;
      const int k = r / NN, j = (r - k * NN) / N;
      key[g] = ((int64_t)(j / B) * N + k) * (int64_t)NN + (r - k * NN);
      ord[g] = (int)g;
    }
    if (env_int("ENPROP_STAGED_ORDER", 1) != 0)  // 0: plain row order (A/B)
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
  }
  sm.n_interior = 0;
  if (interior_lo < interior_hi) {  // interior stages first, each part in sweep order
    auto interior = [&](int g) { return hd[g].R0 >= interior_lo && hd[g].R1 <= interior_hi; };
    const auto mid = std::stable_partition(ord.begin(), ord.end(), interior);
    sm.n_interior = (int)(mid - ord.begin());
  }
  {  // store descriptors and index blocks in sweep order
    std::vector<StageDesc> sorted(hd.size());
    for (size_t q = 0; q < hd.size(); ++q) {
      sorted[q] = hd[ord[q]];
      sorted[q].g = ord[q];
      sorted[q].blk_off = (int64_t)q * idx_bytes;
    }
    hd.swap(sorted);
  }
  sm.s = s;
  sm.N = N;
  sm.tm = tm;
  sm.xlo = xlo;
  sm.xhi = xhi < 0 ? tm.rows : xhi;
  sm.blk_bytes = off;
  sm.idx_bytes = idx_bytes;
  int* bad = nullptr;
  err = cudaMalloc(&sm.desc, hd.size() * sizeof(StageDesc) + 16);

  if (err == cudaSuccess) err = cudaMalloc(&sm.blk, off + 16);
  if (err == cudaSuccess) err = cudaMalloc(&bad, sizeof(int));
  if (err == cudaSuccess) err = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(sm.desc, hd.data(), hd.size() * sizeof(StageDesc), cudaMemcpyHostToDevice, st);
  if (err == cudaSuccess) {
    const int work = sm.nstages * RS;
    k_stage_fill<<<(work + 255) / 256, 256, 0, st>>>(tm, sm.nstages, T, N, L, RS, 8 * s, max_upper, zc,
                                                     idx_bytes, sm.desc, row_map, col_entry, vpos,
                                                     sm.blk, bad);
    err = cudaGetLastError();
  }
  int hbad = 0;
  if (err == cudaSuccess) err = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  if (bad) cudaFree(bad);
  if (err == cudaSuccess && hbad) err = cudaErrorInvalidValue;  // not the structured 27-point graph
  if (err != cudaSuccess) free_stage_map(sm);
  return err;
}

StageMap stage_range(const StageMap& sm, int pos0, int count, int xlo, int xhi) {
  StageMap r = sm;  // a view: desc / blk are not owned (never free_stage_map it)
  r.desc = sm.desc + pos0;
  r.blk = sm.blk + (int64_t)pos0 * sm.idx_bytes;
  r.nstages = count;
  r.blk_bytes = (int64_t)count * sm.idx_bytes;
  r.n_interior = 0;
  r.xlo = xlo;
  r.xhi = xhi;
  return r;
}

void free_stage_map(StageMap& sm) {
  if (sm.desc) cudaFree(sm.desc);
  if (sm.blk) cudaFree(sm.blk);
  sm = StageMap{};
}

// ENPROP_STAGED_CTAS (A/B): 2 = two CTAs per SM with one stage buffer each
// (default at s >= 16: 64^3/s=32 canonical SpMV + fused finalize 0.272 ->
// 0.236 ms, 24-group serial bench 536 -> 545 samples/s), 1 = one CTA per SM
// with two buffers (s = 4 always: its index blocks do not fit twice)
int staged_ctas() {
  static const int v = env_int("ENPROP_STAGED_CTAS", 2) == 1 ? 1 : 2;
  return v;
}

template <int S, int NB>
static cudaError_t cg_spmv_staged_nb(bool tiles, bool fuse_fin, const StageMap& sm, const double* values,
                                     const double* p, double* q, const FinArgs& f, cudaStream_t st) {
  using Sh = StagedShape<S, NB>;
  // per device: SM count, published only after the shared-memory opt-in is
  // done (solves on several host threads launch concurrently)
  static std::atomic<int> sms[64];
  static std::mutex init_mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!sms[dev].load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lock(init_mu);
    if (!sms[dev].load(std::memory_order_relaxed)) {
      int count = 0;
      cudaError_t err = cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(k_cg_spmv_staged<S, true, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM);
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(k_cg_spmv_staged<S, false, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM);
      if (err != cudaSuccess) return err;
      sms[dev].store(count, std::memory_order_release);
    }
  }
  const int slots = sms[dev].load(std::memory_order_acquire) * (NB == 2 ? 1 : 2);  // resident CTAs
  if (sm.nstages == 0) return cudaSuccess;
  const int grid = sm.nstages < slots ? sm.nstages : slots;
  if (tiles)
    // the fused finalize's grid barrier needs every CTA resident: a
    // cooperative launch guarantees it even with other streams' kernels
    // (possibly persistent ones of concurrent sample groups) on the GPU
    launch_kk(2 | (fuse_fin ? kLaunchCooperative : 0), k_cg_spmv_staged<S, true, NB>, dim3(grid), dim3(256), Sh::SMEM, st, sm.tm, sm.N, sm.nstages, sm.xlo, sm.xhi, sm.desc, sm.blk,
                                                           values, p, q, f, fuse_fin ? 1 : 0, staged_pf());
  else
    launch_kk(2, k_cg_spmv_staged<S, false, NB>, dim3(grid), dim3(256), Sh::SMEM, st, sm.tm, sm.N, sm.nstages, sm.xlo, sm.xhi, sm.desc, sm.blk,
                                                            values, p, q, f, 0, staged_pf());
  return cudaGetLastError();
}

template <int S>
static cudaError_t cg_spmv_staged_s(bool tiles, bool fuse_fin, const StageMap& sm, const double* values,
                                    const double* p, double* q, const FinArgs& f, cudaStream_t st) {
  if constexpr (S >= 16)  // s = 4's index blocks do not fit two CTAs per SM
    if (staged_ctas() == 2) return cg_spmv_staged_nb<S, 1>(tiles, fuse_fin, sm, values, p, q, f, st);
  return cg_spmv_staged_nb<S, 2>(tiles, fuse_fin, sm, values, p, q, f, st);
}

cudaError_t launch_cg_spmv_staged(int s, bool tiles, bool fuse_fin, const StageMap& sm,
                                  const double* values, const double* p, double* q, const FinArgs& f,
                                  cudaStream_t st) {
  if (s == 32) return cg_spmv_staged_s<32>(tiles, fuse_fin, sm, values, p, q, f, st);
  if (s == 16) return cg_spmv_staged_s<16>(tiles, fuse_fin, sm, values, p, q, f, st);
  if (s == 4) return cg_spmv_staged_s<4>(tiles, fuse_fin, sm, values, p, q, f, st);
  return cudaErrorInvalidValue;
}

}  // namespace ep
