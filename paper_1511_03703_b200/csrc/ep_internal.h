// Host internals shared by the C-ABI translation units (ep_capi.cu, ep_dist.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "enprop_b200.h"
#include "ep_common.cuh"
#include "ep_kernels.h"

#define EP_CUDA(call)                                  \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

struct enprop_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int* pinned_flags = nullptr;  // [2] convergence flags read back by the CG driver
  cudaEvent_t flag_ev[2] = {nullptr, nullptr};
  int spmv_pipeline = 0;    // ENPROP_OPT_SPMV_PIPELINE
  int fused_direction = 0;  // ENPROP_OPT_FUSED_DIRECTION (split measured faster on B200)
  int symmetric_storage = 1;  // ENPROP_OPT_SYMMETRIC_STORAGE (problems created afterwards)
  int pdl = 0;                // ENPROP_OPT_PDL
  int spmv_variant = -1;      // ENPROP_OPT_SPMV_VARIANT
  int graphs = 1;             // ENPROP_OPT_GRAPHS
  // optional CUDA-event timing of the CG SpMV launches (bench roofline)
  int profile = 0;
  std::vector<cudaEvent_t> prof_ev;  // 5 events per profiled iteration, reused
  size_t prof_used = 0;
  double prof_ms = 0.0;       // CG SpMV kernel (without the direction pass)
  int64_t prof_count = 0;     // profiled iterations that did work
  // spmv phase, fin pq, update, fin rr, iteration, solve, init, loop, early-exit,
  // direction, spmv kernel (enprop_b200.h)
  double prof_detail[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cudaEvent_t prof_solve_ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace ep_internal {

// Installs a context's launch options (ep_common.cuh LaunchOpts) on this host
// thread for the duration of one C-ABI call.
struct ScopedLaunchOpts {
  ep::LaunchOpts saved;
  explicit ScopedLaunchOpts(const enprop_ctx* c) : saved(ep::launch_opts()) {
    if (c) ep::launch_opts() = ep::LaunchOpts{c->pdl, c->spmv_variant};
  }
  ~ScopedLaunchOpts() { ep::launch_opts() = saved; }
};

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* where);
bool valid_width(int s);

// Device tables of one (mesh, field, coefficients) combination.
struct AsmSetup {
  double* F = nullptr;
  ep::AsmTables* tab = nullptr;
  ep::AsmArgs args{};
};
int make_asm_setup(enprop_ctx* c, int n, const enprop_kl_params* kl,
                   const enprop_pde_coeffs* coeffs, AsmSetup& out);
void free_asm_setup(AsmSetup& s);
cudaError_t launch_negate(int64_t n, const double* a, double* b, cudaStream_t st);

}  // namespace ep_internal
