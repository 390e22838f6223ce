// Canonical finalize and the CG scalar phase (device code shared by the
// finalize kernel in ep_kernels.cu and the staged SpMV's fused tail in
// ep_staged.cu).  Reduction order: DESIGN.md §4.
#pragma once
#include "ep_common.cuh"
#include "ep_kernels.h"

namespace ep {

__device__ __forceinline__ int atomic_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// =============================================================================
// CG scalar phases (pcg.hpp:52-103), executed by one thread after the lanes'
// dot products are known.  Coupled solves keep their scalars replicated across
// lanes; uncoupled solves run s independent copies of pcg_solve<double>.
// =============================================================================
// One warp runs the phase; lane e owns sample lane e (e < S). Scalars shared by
// the lanes (it, done, status, coupled reductions) are formed by lane 0 after
// warp votes, so per-lane work (sqrt, divisions) runs in parallel.
template <int S>
__device__ void cg_phase(int phase, const double* lanes, CgState* cg, double* hist,
                         double* lanes_out) {
  const int e = threadIdx.x & 31;
  const bool mine = e < S;
  if (phase == kPhaseNone) {
    if (mine) lanes_out[e] = lanes[e];
    if (e == 0) {
      double acc = 0.0;  // reduce_sum (ensemble.hpp:240-244)
      for (int k = 0; k < S; ++k) acc = EP_DADD(acc, lanes[k]);
      lanes_out[S] = acc;
    }
    return;
  }
  const double tol = cg->tol;
  const int maxit = cg->maxit;
  const int it0 = cg->it;
  // Deferred x updates: RR records which lanes updated r (and so owe
  // x += alpha*p); the next direction pass pays them, so PQ clears the record.
  const int was_active = mine ? cg->active[e] : 0;
  if (mine) cg->pending[e] = phase == kPhaseRR ? was_active : 0;
  if (cg->flavour == 0) {  // ---------------------------------------------- coupled
    double d = 0.0;  // reduce_sum over lanes, left to right
#pragma unroll 1
    for (int k = 0; k < S; ++k) d = EP_DADD(d, lanes[k]);
    if (phase == kPhaseInit) {  // b_norm = norm2(b); r = b; p = z = r; rz = dot(r, z)
      const double bn = sqrt(d);
      if (e == 0) {
        cg->it = 0;
        cg->bnorm[0] = bn;
        cg->status = 0;
        cg->iters[0] = 0;
      }
      if (bn == 0.0) {  // pcg.hpp:62-66
        if (e == 0) {
          hist[0] = 0.0;
          cg->hist_len[0] = 1;
          cg->done = 1;
        }
        return;
      }
      if (mine) cg->rz[e] = d;
      const double rel = sqrt(d) / bn;
      int done = 0;
      if (rel < tol) done = 1;
      else if (0 >= maxit) done = 2;
      if (e == 0) {
        hist[0] = rel;
        cg->hist_len[0] = 1;
        if (done == 2) cg->status = 2;
        cg->done = done ? 1 : 0;
      }
      if (mine) cg->active[e] = done ? 0 : 1;
    } else if (phase == kPhasePQ) {  // pq = dot(p, q); alpha = rz / pq
      if (d <= 0.0) {
        if (e == 0) {
          cg->status = 3;
          cg->iters[0] = it0;
          cg->done = 1;
        }
        return;
      }
      const double alpha = cg->rz[0] / d;
      if (mine) cg->alpha[e] = alpha;
    } else {  // kPhaseRR: rz_next = dot(r, z); beta; next relative residual
      const double beta = d / cg->rz[0];
      const int it = it0 + 1;
      const double rel = sqrt(d) / cg->bnorm[0];
      __syncwarp();  // every lane has read rz[0] before it is replaced
      if (mine) {
        cg->beta[e] = beta;
        cg->rz[e] = d;
      }
      if (e == 0) {
        cg->it = it;
        hist[it] = rel;
        cg->hist_len[0] = it + 1;
        if (rel < tol) {
          cg->iters[0] = it;
          cg->done = 1;
        } else if (it >= maxit) {
          cg->iters[0] = it;
          cg->status = 2;
          cg->done = 1;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------ uncoupled
  int st = 0, act = 0;
  if (phase == kPhaseInit) {
    if (mine) {
      const double d = lanes[e];
      const double bn = sqrt(d);
      cg->bnorm[e] = bn;
      cg->iters[e] = 0;
      cg->hist_len[e] = 1;
      if (bn == 0.0) {
        hist[e] = 0.0;
      } else {
        cg->rz[e] = d;
        const double rel = sqrt(d) / bn;
        hist[e] = rel;
        if (rel < tol) {
        } else if (0 >= maxit) {
          st = 2;
        } else {
          act = 1;
        }
      }
      cg->lane_status[e] = st;
      cg->active[e] = act;
    }
    const int any = __any_sync(0xffffffffu, act);
    const int worst = __reduce_max_sync(0xffffffffu, st);
    if (e == 0) {
      cg->it = 0;
      cg->status = worst;
      cg->done = !any;
    }
  } else if (phase == kPhasePQ) {
    if (mine && was_active) {
      const double d = lanes[e];
      if (d <= 0.0) {
        cg->lane_status[e] = 3;
        cg->iters[e] = it0;
        cg->active[e] = 0;
        st = 3;
      } else {
        cg->alpha[e] = cg->rz[e] / d;
        act = 1;
      }
    }
    const int any = __any_sync(0xffffffffu, act);
    const int worst = __reduce_max_sync(0xffffffffu, st);
    if (e == 0) {
      if (worst > cg->status) cg->status = worst;
      if (!any) cg->done = 1;
    }
  } else {
    const int it = it0 + 1;
    if (mine && was_active) {
      const double d = lanes[e];
      cg->beta[e] = d / cg->rz[e];
      cg->rz[e] = d;
      const double rel = sqrt(d) / cg->bnorm[e];
      hist[(size_t)it * S + e] = rel;
      cg->hist_len[e] = it + 1;
      if (rel < tol) {
        cg->iters[e] = it;
        cg->active[e] = 0;
      } else if (it >= maxit) {
        cg->iters[e] = it;
        cg->lane_status[e] = 2;
        cg->active[e] = 0;
        st = 2;
      } else {
        act = 1;
      }
    }
    const int any = __any_sync(0xffffffffu, act);
    const int worst = __reduce_max_sync(0xffffffffu, st);
    if (e == 0) {
      cg->it = it;
      if (worst > cg->status) cg->status = worst;
      if (!any) cg->done = 1;
    }
  }
}

// Canonical finalize of one segment by one 256-thread CTA. Thread (block b,
// sample e) folds the block's kBlockTiles tile partials in registers
// (v[i] += v[i+h], h = 8..1; missing tiles are +0.0) -- a warp covers 32
// consecutive samples, so every load is one coalesced row of partials, and a
// thread's kFinItems blocks are loaded together -- and thread e then forms the
// segment sum 0.0 + block_0 + block_1 + ... from shared memory (sblk).
constexpr int kFinThreads = 256;
constexpr int kFinItems = 3;   // (block, sample) items per thread per round
constexpr int kFinItems2 = 12;  // (segment, sample) items per thread per round (total)

template <int S>
struct FinShape {
  static constexpr int CHUNK = kFinThreads * kFinItems / S;    // blocks per round
  static constexpr int CHUNK2 = kFinThreads * kFinItems2 / S;  // segments per round
};

template <int S>
__device__ __forceinline__ void fin_segment_fold(const TileMap& tm, const FinArgs& f, int seg,
                                                 double* sblk) {
  constexpr int CHUNK = FinShape<S>::CHUNK;
  const int ntiles = tm.tiles_in_seg(seg);
  const int nblk = (ntiles + kBlockTiles - 1) / kBlockTiles;
  const double* part = f.partials + (size_t)seg * tm.tiles_per_seg * S;
  double acc = 0.0;
  for (int b0 = 0; b0 < nblk; b0 += CHUNK) {
    const int cnt = min(CHUNK, nblk - b0);
    double v[kFinItems][kBlockTiles];
#pragma unroll
    for (int it = 0; it < kFinItems; ++it) {
      const int idx = threadIdx.x + it * kFinThreads;
      const int b = idx / S, e = idx - b * S;
      const int t0 = (b0 + b) * kBlockTiles;
      const bool ok = idx < cnt * S;
#pragma unroll
      for (int i = 0; i < kBlockTiles; ++i)
        v[it][i] = ok && t0 + i < ntiles ? __ldcg(part + (size_t)(t0 + i) * S + e) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < kFinItems; ++it) {
#pragma unroll
      for (int h = kBlockTiles / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int i = 0; i < h; ++i) v[it][i] = EP_DADD(v[it][i], v[it][i + h]);
      const int idx = threadIdx.x + it * kFinThreads;
      if (idx < cnt * S) sblk[idx] = v[it][0];
    }
    __syncthreads();
    if (threadIdx.x < S) {
#pragma unroll 8
      for (int b = 0; b < cnt; ++b) acc = EP_DADD(acc, sblk[b * S + threadIdx.x]);
    }
    __syncthreads();
  }
  if (threadIdx.x < S) {
    f.seg_sums[(size_t)seg * S + threadIdx.x] = acc;
    __threadfence();  // before the arrival (fin_total_phase / grid barrier) of another thread
  }
}

// After a CTA's segment folds: the last CTA to arrive (acq_rel counter,
// self-resetting) forms 0.0 + seg_0 + seg_1 + ... per lane (stot scratch) and
// warp 0 runs the CG phase. Every thread of the CTA must call it.
template <int S>
__device__ __forceinline__ void fin_total_phase(const TileMap& tm, const FinArgs& f, double* stot,
                                                double* lanes, int* s_final, int arrivals = 1) {
  constexpr int CHUNK2 = FinShape<S>::CHUNK2;
  __syncthreads();
  if (threadIdx.x == 0)
    *s_final = (atomic_add_acq_rel_gpu(f.seg_done, arrivals) + arrivals == tm.num_segs);
  __syncthreads();
  if (!*s_final) return;
  double tot = 0.0;
  for (int k0 = 0; k0 < tm.num_segs; k0 += CHUNK2) {
    const int cnt = min(CHUNK2, tm.num_segs - k0);
    double w[kFinItems2];
#pragma unroll
    for (int it = 0; it < kFinItems2; ++it) {
      const int idx = threadIdx.x + it * kFinThreads;
      w[it] = idx < cnt * S ? __ldcg(f.seg_sums + (size_t)k0 * S + idx) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < kFinItems2; ++it) {
      const int idx = threadIdx.x + it * kFinThreads;
      if (idx < cnt * S) stot[idx] = w[it];
    }
    __syncthreads();
    if (threadIdx.x < S) {
#pragma unroll 8
      for (int k = 0; k < cnt; ++k) tot = EP_DADD(tot, stot[k * S + threadIdx.x]);
    }
    __syncthreads();
  }
  if (threadIdx.x < S) lanes[threadIdx.x] = tot;
  __syncthreads();
  if (threadIdx.x == 0) *f.seg_done = 0;
  if (threadIdx.x < 32) cg_phase<S>(f.phase, lanes, f.cg, f.hist, f.lanes_out);
}

}  // namespace ep
