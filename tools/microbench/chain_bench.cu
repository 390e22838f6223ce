// Microbenchmark of the serial dot chain (ep_chain.cu design space): one warp,
// lane e = sample e, acc += x[row][e] over `rows` rows; loads run DEPTH batches
// of 16 rows ahead in registers; optional TMA L2 prefetch AHEAD rows ahead.
// Prints ms and cycles per row for load flavours / depths / prefetch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o chain_bench chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  if constexpr (MODE == 0) return __ldcg(p);
  else if constexpr (MODE == 1) return __ldg(p);
  else if constexpr (MODE == 2) return *p;
  else {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
  }
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int S, int DEPTH, int MODE, int PF>
__global__ void __launch_bounds__(32, 1) chain(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  constexpr int B = 16;
  const int e = threadIdx.x;
  const int el = e < S ? e : 0;
  const double* pu = u + el;
  const int nfull = rows / B;
  double a[DEPTH][B];
  long long t0 = clock64();
  if (PF) for (int r0 = 0; r0 < PF; r0 += 64) if (e == 0) prefetch_l2(u + (size_t)r0 * S, 64 * 8 * S);
#pragma unroll
  for (int d = 0; d + 1 < DEPTH; ++d)
#pragma unroll
    for (int k = 0; k < B; ++k) a[d][k] = ld<MODE>(pu + ((size_t)d * B + k) * S);
  double acc = 0.0;
  for (int b0 = 0; b0 < nfull; b0 += DEPTH) {
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const int bt = b0 + j;
      if (bt < nfull) {
        const int nb = bt + DEPTH - 1;
        if (nb < nfull) {
#pragma unroll
          for (int k = 0; k < B; ++k) a[(j + DEPTH - 1) % DEPTH][k] = ld<MODE>(pu + ((size_t)nb * B + k) * S);
        }
        if (PF && (bt * B) % 64 == 0 && e == 0 && bt * B + PF + 64 <= rows)
          prefetch_l2(u + (size_t)(bt * B + PF) * S, 64 * 8 * S);
#pragma unroll
        for (int k = 0; k < B; ++k) acc = __dadd_rn(acc, a[j][k]);
      }
    }
  }
  long long t1 = clock64();
  out[e] = acc;
  if (e == 0) cyc[0] = t1 - t0;
}

__global__ void pure_chain(int n, double* out, long long* cyc, double a) {
  double acc = 0.0, x[16];
  for (int k = 0; k < 16; ++k) x[k] = a * k;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 16)
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = __dadd_rn(acc, x[k]);
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


// ---- shared-memory ring variants -------------------------------------------
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// TMA (cp.async.bulk) ring: NST stages of SB bytes, mbarrier per stage; one warp
// (lane 0 issues the refills), LPR lanes per row part: this CTA handles samples
// [part*SP, part*SP + SP) of S (SP = S / PARTS) -- PARTS > 1 uses cp.async (16 B).
template <int S, int SB, int NST, int PF>
__global__ void __launch_bounds__(32, 1) ring_tma(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bar[NST];
  constexpr int R = SB / (8 * S);
  const int e = threadIdx.x, el = e < S ? e : 0;
  const int nst = rows / R;
  if (e == 0) {
    for (int k = 0; k < NST; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  long long t0 = clock64();
  auto issue = [&](int c) {
    if (e == 0 && c < nst) {
      const int slot = c % NST;
      if (PF && (c * R) % 64 == 0 && c * R + PF + 64 <= rows)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)(c * R + PF) * S), "r"(64 * 8 * S) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(SB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + slot * SB)),
                   "l"(u + (size_t)c * R * S), "r"(SB), "r"(su32(&bar[slot])) : "memory");
    }
  };
  for (int c = 0; c < NST; ++c) issue(c);
  double acc = 0.0;
  for (int c = 0; c < nst; ++c) {
    const int slot = c % NST;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar[slot])), "r"((c / NST) & 1) : "memory");
    const double* a = reinterpret_cast<const double*>(sm + slot * SB) + el;
#pragma unroll
    for (int k = 0; k < R; ++k) acc = __dadd_rn(acc, a[k * S]);
    __syncwarp();
    issue(c + NST);
  }
  long long t1 = clock64();
  out[e] = acc;
  if (e == 0) cyc[0] = t1 - t0;
}

// cp.async (16 B per lane) ring with commit/wait_group ordering; the CTA covers
// SP samples (SP*8 bytes of each S*8-byte row, at column offset part*SP).
template <int S, int SP, int SB, int NST, int PF>
__global__ void __launch_bounds__(32, 1) ring_cpa(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int RB = SP * 8;           // bytes per row part
  constexpr int R = SB / RB;           // rows per stage
  constexpr int PER = SB / 16 / 32;    // 16-B copies per lane per stage
  static_assert(PER >= 1, "stage too small");
  const int e = threadIdx.x, el = e < SP ? e : 0;
  const int part = blockIdx.x;
  const int nst = rows / R;
  long long t0 = clock64();
  auto issue = [&](int c) {
    if (c < nst) {
      const int slot = c % NST;
      if (PF && e == 0 && (c * R) % 64 == 0 && c * R + PF + 64 <= rows)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)(c * R + PF) * S), "r"(64 * 8 * S) : "memory");
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int idx = q * 32 + e;           // 16-B granule of the stage
        const int r = idx / (RB / 16), g = idx % (RB / 16);
        const char* src = reinterpret_cast<const char*>(u + (size_t)(c * R + r) * S + part * SP) + g * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + slot * SB + idx * 16)), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int c = 0; c < NST - 1; ++c) issue(c);
  double acc = 0.0;
  for (int c = 0; c < nst; ++c) {
    issue(c + NST - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
    __syncwarp();
    const double* a = reinterpret_cast<const double*>(sm + (c % NST) * SB) + el;
#pragma unroll
    for (int k = 0; k < R; ++k) acc = __dadd_rn(acc, a[k * SP]);
    __syncwarp();
  }
  long long t1 = clock64();
  out[part * 32 + e] = acc;
  if (e == 0 && part == 0) cyc[0] = t1 - t0;
}

// Two warps: warp 1 lane 0 produces (TMA ring, waits on `empty`), warp 0
// consumes with the next stage's LDS and the stage-after-next's barrier probe
// issued BEFORE the current stage's DADD chain, so their latencies overlap it.
template <int S, int SB, int NST, int PF, int TEST>
__global__ void __launch_bounds__(64, 1) ring2(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long full[NST], empty[NST];
  constexpr int R = SB / (8 * S);
  const int e = threadIdx.x & 31;
  const int el = e < S ? e : 0;
  const int nst = rows / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[k])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[k])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    for (int c = 0; c < nst; ++c) {
      const int slot = c % NST;
      if (c >= NST)
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&empty[slot])), "r"(((c / NST) - 1) & 1) : "memory");
      if (PF && (c * R) % 64 == 0 && c * R + PF + 64 <= rows)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)(c * R + PF) * S), "r"(64 * 8 * S) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(SB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + slot * SB)),
                   "l"(u + (size_t)c * R * S), "r"(SB), "r"(su32(&full[slot])) : "memory");
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  auto probe = [&](int c) -> unsigned {
    unsigned ok;
    if constexpr (TEST)
      asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su32(&full[c % NST])), "r"((c / NST) & 1) : "memory");
    else
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su32(&full[c % NST])), "r"((c / NST) & 1) : "memory");
    return ok;
  };
  auto wait = [&](int c) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&full[c % NST])), "r"((c / NST) & 1) : "memory");
  };
  long long t0 = clock64();
  double cur[R], nxt[R];
  if (nst > 0) wait(0);
  if (nst > 1) wait(1);
  {
    const double* a = reinterpret_cast<const double*>(sm) + el;
#pragma unroll
    for (int k = 0; k < R; ++k) cur[k] = a[k * S];
  }
  double acc = 0.0;
  for (int c = 0; c < nst; ++c) {
    if (c + 1 < nst) {
      const double* a = reinterpret_cast<const double*>(sm + ((c + 1) % NST) * SB) + el;
#pragma unroll
      for (int k = 0; k < R; ++k) nxt[k] = a[k * S];
    }
    const unsigned tok = c + 2 < nst ? probe(c + 2) : 1u;
#pragma unroll
    for (int k = 0; k < R; ++k) acc = __dadd_rn(acc, cur[k]);
    __syncwarp();
    if (e == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[c % NST])) : "memory");
    if (!tok) wait(c + 2);
#pragma unroll
    for (int k = 0; k < R; ++k) cur[k] = nxt[k];
  }
  long long t1 = clock64();
  out[e] = acc;
  if (e == 0) cyc[0] = t1 - t0;
}

// r3: the consumer never executes an mbarrier op. Warp 1 lane 0 waits on the
// TMA barriers and publishes `ready` (stages landed) in shared memory; warp 0
// publishes `consumed`. Both counters are plain volatile shared words.
template <int S, int SB, int NST, int PF>
__global__ void __launch_bounds__(64, 1) ring3(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long full[NST];
  __shared__ volatile int ready, consumed;
  constexpr int R = SB / (8 * S);
  const int e = threadIdx.x & 31;
  const int el = e < S ? e : 0;
  const int nst = rows / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ready = 0;
    consumed = 0;
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    int issued = 0;
    for (int c = 0; c < nst; ++c) {
      // keep NST stages in flight: issue while slots are free (at least up to
      // stage c, waiting for the consumer to free a slot), then retire stage c
      while (issued < nst && (issued <= c || issued < consumed + NST)) {
        while (issued >= consumed + NST) {}
        const int slot = issued % NST;
        if (PF && (issued * R) % 64 == 0 && issued * R + PF + 64 <= rows)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(u + (size_t)(issued * R + PF) * S), "r"(64 * 8 * S) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + slot * SB)),
                     "l"(u + (size_t)issued * R * S), "r"(SB), "r"(su32(&full[slot])) : "memory");
        ++issued;
      }
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&full[c % NST])), "r"((c / NST) & 1) : "memory");
      __threadfence_block();
      ready = c + 1;
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  double cur[R], nxt[R];
  while (ready < (nst > 1 ? 2 : nst)) {}
  __threadfence_block();
  {
    const double* a = reinterpret_cast<const double*>(sm) + el;
#pragma unroll
    for (int k = 0; k < R; ++k) cur[k] = a[k * S];
  }
  double acc = 0.0;
  for (int c = 0; c < nst; ++c) {
    if (c + 1 < nst) {
      const double* a = reinterpret_cast<const double*>(sm + ((c + 1) % NST) * SB) + el;
#pragma unroll
      for (int k = 0; k < R; ++k) nxt[k] = a[k * S];
    }
    const int rd = ready;  // early: consumed after the chain
#pragma unroll
    for (int k = 0; k < R / 2; ++k) acc = __dadd_rn(acc, cur[k]);
    if (e == 0) consumed = c + 1;  // slot c: its values are in registers (cur) by now
#pragma unroll
    for (int k = R / 2; k < R; ++k) acc = __dadd_rn(acc, cur[k]);
    if (c + 2 < nst && rd < c + 3) {
      while (ready < c + 3) {}
    }
    __threadfence_block();
#pragma unroll
    for (int k = 0; k < R; ++k) cur[k] = nxt[k];
  }
  long long t1 = clock64();
  out[e] = acc;
  if (e == 0) cyc[0] = t1 - t0;
}

// latency of one TMA bulk copy (SB bytes) to completion observed by try_wait
__global__ void tma_lat(const double* u, long long* cyc, int bytes, int stride) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bar;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  long long tot = 0;
  for (int i = 0; i < 32; ++i) {
    long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm)),
                 "l"((const char*)u + (size_t)i * stride), "r"(bytes), "r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar)), "r"(i & 1) : "memory");
    tot += clock64() - t0;
  }
  cyc[0] = tot / 32;
}

// ring4: warp 1 lane 0 produces (waits `empty`, issues TMA); warp 0 waits
// `full`, then reads the stage in 16-row register batches (next batch's LDS
// issued before the current batch's DADDs) and arrives on `empty`.
template <int S, int SB, int NST>
__global__ void __launch_bounds__(64, 1) ring4(int rows, const double* __restrict__ u, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long full[NST], empty[NST];
  constexpr int R = SB / (8 * S);
  constexpr int B = 16;
  const int e = threadIdx.x & 31;
  const int el = e < S ? e : 0;
  const int nst = rows / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[k])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[k])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    for (int c = 0; c < nst; ++c) {
      const int slot = c % NST;
      if (c >= NST)
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&empty[slot])), "r"(((c / NST) - 1) & 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(SB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + slot * SB)),
                   "l"(u + (size_t)c * R * S), "r"(SB), "r"(su32(&full[slot])) : "memory");
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  double acc = 0.0;
  double cur[B], nxt[B];
  for (int c = 0; c < nst; ++c) {
    const int slot = c % NST;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(&full[slot])), "r"((c / NST) & 1) : "memory");
    const double* a = reinterpret_cast<const double*>(sm + slot * SB) + el;
#pragma unroll
    for (int k = 0; k < B; ++k) cur[k] = a[k * S];
#pragma unroll 1
    for (int b = 0; b < R / B; ++b) {
      if (b + 1 < R / B) {
#pragma unroll
        for (int k = 0; k < B; ++k) nxt[k] = a[((b + 1) * B + k) * S];
      }
#pragma unroll
      for (int k = 0; k < B; ++k) acc = __dadd_rn(acc, cur[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) cur[k] = nxt[k];
    }
    __syncwarp();
    if (e == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
  }
  long long t1 = clock64();
  out[e] = acc;
  if (e == 0) cyc[0] = t1 - t0;
}

template <typename K>
void timek(const char* name, K kern, int grid, int smem, int rows, const double* u, double* out, long long* cyc) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, 32, smem>>>(rows, u, out, cyc);
  cudaEventRecord(e0);
  kern<<<grid, 32, smem>>>(rows, u, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s rows=%d: %.3f ms, %.2f cycles/row  (%s)\n", name, rows, ms, (double)h / rows,
         cudaGetErrorString(cudaGetLastError()));
}

template <int S, int DEPTH, int MODE, int PF>
void run(const char* name, int rows, const double* u, double* out, long long* cyc) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chain<S, DEPTH, MODE, PF><<<1, 32>>>(rows, u, out, cyc);
  // flush L2 between reps by touching a big buffer is done by caller ordering
  cudaEventRecord(e0);
  chain<S, DEPTH, MODE, PF><<<1, 32>>>(rows, u, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s S=%2d rows=%d: %.3f ms, %.2f cycles/row\n", name, S, rows, ms, (double)h / rows);
}

template <typename K>
void timek2(const char* name, K kern, int smem, int rows, const double* u, double* out, long long* cyc) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<1, 64, smem>>>(rows, u, out, cyc);
  cudaEventRecord(e0);
  kern<<<1, 64, smem>>>(rows, u, out, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s rows=%d: %.3f ms, %.2f cycles/row  (%s)\n", name, rows, ms, (double)h / rows,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int rows = 274625;
  double *u, *out, *flush;
  long long* cyc;
  cudaMalloc(&u, (size_t)rows * 32 * 8);
  cudaMemset(u, 0, (size_t)rows * 32 * 8);
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  const size_t fb = (size_t)512 << 20;
  cudaMalloc(&flush, fb);
  pure_chain<<<1, 32>>>(1 << 20, out, cyc, 1e-9);
  long long h;
  cudaDeviceSynchronize();
  pure_chain<<<1, 32>>>(1 << 20, out, cyc, 1e-9);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pure register DADD chain: %.2f cycles/add\n", (double)h / (1 << 20));
  // second launch of each run reads the data warm in L2 when it fits (S=1: 2 MB)
#define R(S, D, M, P) run<S, D, M, P>(#S " D" #D " M" #M " PF" #P, rows, u, out, cyc)
  R(1, 4, 0, 0); R(1, 4, 1, 0); R(1, 4, 3, 0); R(1, 8, 0, 0);
  R(32, 2, 0, 0); R(32, 4, 0, 0); R(32, 6, 0, 0); R(32, 4, 1, 0); R(32, 4, 3, 0);
  R(32, 4, 0, 512); R(32, 4, 0, 1024); R(32, 4, 0, 2048); R(32, 6, 3, 1024); R(32, 4, 3, 2048);
  R(8, 4, 0, 0); R(8, 4, 0, 1024);
  // big array (> L2) for the streamed case: 64^3 rows x 32 = 70 MB fits L2; use 4x rows
  const int big = 4 * rows;
  double* ub;
  cudaMalloc(&ub, (size_t)big * 32 * 8);
  cudaMemset(ub, 0, (size_t)big * 32 * 8);
#define T(NAME, K, G, SM) timek(NAME, K, G, SM, rows, u, out, cyc); timek(NAME " [big]", K, G, SM, big, ub, out, cyc)
#define T2(NAME, K, SM) timek2(NAME, K, SM, rows, u, out, cyc); timek2(NAME " [big]", K, SM, big, ub, out, cyc)
  for (int b : {2048, 4096, 16384}) for (int st : {4096, 1 << 20}) {
    cudaFuncSetAttribute(tma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    tma_lat<<<1, 1, 16384>>>(ub, cyc, b, st);
    long long hh; cudaMemcpy(&hh, cyc, 8, cudaMemcpyDeviceToHost);
    printf("TMA %5d B copy latency (stride %d): %lld cycles\n", b, st, hh);
  }
  T2("r4 S32 16KBx8", (ring4<32, 16384, 8>), 16384 * 8);
  T2("r4 S32 32KBx6", (ring4<32, 32768, 6>), 32768 * 6);
  T2("r4 S32 32KBx4", (ring4<32, 32768, 4>), 32768 * 4);
  T2("r4 S32 16KBx12", (ring4<32, 16384, 12>), 16384 * 12);
  T2("r4 S32 8KBx16", (ring4<32, 8192, 16>), 8192 * 16);
  T2("r4 S16 16KBx8", (ring4<16, 16384, 8>), 16384 * 8);
  T2("r4 S8 16KBx8", (ring4<8, 16384, 8>), 16384 * 8);
  T2("r4 S1 16KBx8", (ring4<1, 16384, 8>), 16384 * 8);
  T2("r3 S32 2KBx6", (ring3<32, 2048, 6, 0>), 2048 * 6);
  T2("r3 S32 2KBx6 pf1024", (ring3<32, 2048, 6, 1024>), 2048 * 6);
  T2("r3 S32 4KBx3 pf1024", (ring3<32, 4096, 3, 1024>), 4096 * 3);
  T2("r3 S32 4KBx3", (ring3<32, 4096, 3, 0>), 4096 * 3);
  T2("r3 S32 2KBx7 pf2048", (ring3<32, 2048, 7, 2048>), 2048 * 7);
  T2("r3 S32 4KBx8", (ring3<32, 4096, 8, 0>), 4096 * 8);
  T2("r3 S32 8KBx8", (ring3<32, 8192, 8, 0>), 8192 * 8);
  T2("r3 S16 2KBx6 pf1024", (ring3<16, 2048, 6, 1024>), 2048 * 6);
  T2("r3 S8 2KBx6 pf1024", (ring3<8, 2048, 6, 1024>), 2048 * 6);
  T2("r3 S4 1KBx12", (ring3<4, 1024, 12, 0>), 1024 * 12);
  T2("r3 S1 256x24", (ring3<1, 256, 24, 0>), 256 * 24);
  T2("r2 S32 4KBx3", (ring2<32, 4096, 3, 0, 0>), 4096 * 3);
  T2("r2 S32 4KBx3 test", (ring2<32, 4096, 3, 0, 1>), 4096 * 3);
  T2("r2 S32 4KBx3 pf1024", (ring2<32, 4096, 3, 1024, 0>), 4096 * 3);
  T2("r2 S32 2KBx6", (ring2<32, 2048, 6, 0, 0>), 2048 * 6);
  T2("r2 S32 2KBx6 pf1024", (ring2<32, 2048, 6, 1024, 0>), 2048 * 6);
  T2("r2 S32 2KBx7 pf2048", (ring2<32, 2048, 7, 2048, 0>), 2048 * 7);
  T2("r2 S32 4KBx4", (ring2<32, 4096, 4, 0, 0>), 4096 * 4);
  T2("r2 S32 4KBx8", (ring2<32, 4096, 8, 0, 0>), 4096 * 8);
  T2("r2 S32 8KBx8", (ring2<32, 8192, 8, 0, 0>), 8192 * 8);
  T2("r2 S16 2KBx6 pf1024", (ring2<16, 2048, 6, 1024, 0>), 2048 * 6);
  T2("r2 S8 2KBx6 pf1024", (ring2<8, 2048, 6, 1024, 0>), 2048 * 6);
  T2("r2 S4 2KBx6", (ring2<4, 2048, 6, 0, 0>), 2048 * 6);
  T2("r2 S1 1KBx6", (ring2<1, 1024, 6, 0, 0>), 1024 * 6);
  T("tma S32 2KB x7", (ring_tma<32, 2048, 7, 0>), 1, 2048 * 7);
  T("tma S32 2KB x7 pf1024", (ring_tma<32, 2048, 7, 1024>), 1, 2048 * 7);
  T("tma S32 4KB x3 pf1024", (ring_tma<32, 4096, 3, 1024>), 1, 4096 * 3);
  T("tma S32 4KB x8", (ring_tma<32, 4096, 8, 0>), 1, 4096 * 8);
  T("tma S32 8KB x8", (ring_tma<32, 8192, 8, 0>), 1, 8192 * 8);
  T("tma S32 16KB x8", (ring_tma<32, 16384, 8, 0>), 1, 16384 * 8);
  T("tma S32 16KB x8 pf2048", (ring_tma<32, 16384, 8, 2048>), 1, 16384 * 8);
  T("tma S1 2KB x7", (ring_tma<1, 2048, 7, 0>), 1, 2048 * 7);
  T("cpa S32 full 2KB x7", (ring_cpa<32, 32, 2048, 7, 0>), 1, 2048 * 7);
  T("cpa S32 full 2KB x7 pf1024", (ring_cpa<32, 32, 2048, 7, 1024>), 1, 2048 * 7);
  T("cpa S32 half 2KB x7 (2 CTAs)", (ring_cpa<32, 16, 2048, 7, 0>), 2, 2048 * 7);
  T("cpa S32 half 2KB x7 pf1024 (2 CTAs)", (ring_cpa<32, 16, 2048, 7, 1024>), 2, 2048 * 7);
  T("cpa S32 quarter 1KB x14 pf1024 (4 CTAs)", (ring_cpa<32, 8, 1024, 14, 1024>), 4, 1024 * 14);
  return 0;
}
