// Host-side setup shared by the C ABI: KL field eigen-structure and the
// sample-independent assembly tables, computed in the reference's exact
// floating-point order (this file is compiled with -ffp-contract=off).
#pragma once
#include <vector>

#include "ep_kernels.h"

namespace ep {

constexpr int kMaxTermsHost = 64;  // AsmArgs carries at most 64 modes

struct KlHost {
  int m = 0;
  double mean = 1.0, sigma = 0.0, corr_length = 1.0;
  std::vector<double> axis_freq, axis_eig, axis_invnorm;
  std::vector<int> axis_cos;
  std::vector<int> mode_axes;  // [m][3]
  std::vector<double> mode_eig, mode_sqrt_eig;
};

// KlField(num_terms, mean, sigma, L): proj/src/kl.cpp:41-89. Returns false on
// invalid parameters (the reference throws std::invalid_argument).
bool kl_init(KlHost& f, int m, double mean, double sigma, double corr_length);
// AxisMode::evaluate (kl.hpp:24-27)
double kl_axis_eval(const KlHost& f, int t, double x);
// Per-axis-mode tables F[t][2c + b] = f_t((c + off_b) * h) for the 2x2x2 Gauss
// offsets off_b = 0.5*(-+1/sqrt(3) + 1.0) (fem.hpp:82-85) and h = 1/n.
std::vector<double> kl_axis_tables(const KlHost& f, int n);
// Sample-independent assembly tables for mesh n (fem.hpp:76-98, 133-191).
void make_asm_tables(AsmTables& t, int n, double alpha, double beta, const double velocity[3]);

}  // namespace ep
