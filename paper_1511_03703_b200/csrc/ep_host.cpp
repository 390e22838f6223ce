// Host setup restated from the reference (see ep_host.h). Compiled with
// -ffp-contract=off so every product/sum rounds exactly as in the reference
// build (proj/CMakeLists.txt:14); std::cos/std::sin/std::sqrt are the same
// glibc routines the reference calls, evaluated on the same arguments.
#include "ep_host.h"

#include <algorithm>
#include <array>
#include <cmath>

namespace ep {

namespace {

constexpr double kPi = 3.14159265358979323846;

// kl.cpp:13-19 (product forms of the two transcendental branch equations)
double branch_residual(double w, double c, bool cosine) {
  return cosine ? w * std::sin(0.5 * w) - c * std::cos(0.5 * w)
                : c * std::sin(0.5 * w) + w * std::cos(0.5 * w);
}

// kl.cpp:21-35: bisection to an interval width of 1e-12
double bisect(double lo, double hi, double c, bool cosine) {
  double flo = branch_residual(lo, c, cosine);
  while (hi - lo > 1e-12) {
    const double mid = 0.5 * (lo + hi);
    const double fmid = branch_residual(mid, c, cosine);
    if ((flo < 0.0) == (fmid < 0.0)) {
      lo = mid;
      flo = fmid;
    } else {
      hi = mid;
    }
  }
  return 0.5 * (lo + hi);
}

struct Candidate {
  std::array<int, 3> axis;
  double eig;
  double sq;
};

}  // namespace

bool kl_init(KlHost& f, int m, double mean, double sigma, double corr_length) {
  if (m < 1 || m > kMaxTermsHost || !(mean > 0.0) || sigma < 0.0 || !(corr_length > 0.0))
    return false;
  f = KlHost{};
  f.m = m;
  f.mean = mean;
  f.sigma = sigma;
  f.corr_length = corr_length;
  const double c = 1.0 / corr_length;
  f.axis_freq.resize(m);
  f.axis_eig.resize(m);
  f.axis_invnorm.resize(m);
  f.axis_cos.resize(m);
  for (int t = 0; t < m; ++t) {  // kl.cpp:47-61
    const int k = t / 2;
    const bool cosine = (t % 2 == 0);
    const double lo = cosine ? 2 * k * kPi : (2 * k + 1) * kPi;
    const double w = bisect(lo, lo + kPi, c, cosine);
    f.axis_cos[t] = cosine ? 1 : 0;
    f.axis_freq[t] = w;
    f.axis_eig[t] = 2.0 * c / (w * w + c * c);
    const double half_sinc = std::sin(w) / (2.0 * w);
    f.axis_invnorm[t] = 1.0 / std::sqrt(cosine ? 0.5 + half_sinc : 0.5 - half_sinc);
  }
  std::vector<Candidate> cand;  // kl.cpp:75-88
  cand.reserve((size_t)m * m * m);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b)
      for (int d = 0; d < m; ++d) {
        const double lambda = f.axis_eig[a] * f.axis_eig[b] * f.axis_eig[d];
        cand.push_back({{a, b, d}, lambda, std::sqrt(lambda)});
      }
  std::sort(cand.begin(), cand.end(), [](const Candidate& p, const Candidate& q) {
    if (p.eig != q.eig) return p.eig > q.eig;
    return p.axis < q.axis;
  });
  f.mode_axes.resize((size_t)m * 3);
  f.mode_eig.resize(m);
  f.mode_sqrt_eig.resize(m);
  for (int i = 0; i < m; ++i) {
    for (int a = 0; a < 3; ++a) f.mode_axes[i * 3 + a] = cand[i].axis[a];
    f.mode_eig[i] = cand[i].eig;
    f.mode_sqrt_eig[i] = cand[i].sq;
  }
  return true;
}

double kl_axis_eval(const KlHost& f, int t, double x) {
  const double arg = f.axis_freq[t] * (x - 0.5);
  return (f.axis_cos[t] ? std::cos(arg) : std::sin(arg)) * f.axis_invnorm[t];
}

std::vector<double> kl_axis_tables(const KlHost& f, int n) {
  const double g = 1.0 / std::sqrt(3.0);
  const double off[2] = {0.5 * (-g + 1.0), 0.5 * (g + 1.0)};  // fem.hpp:84-85
  const double h = 1.0 / n;                                    // mesh.hpp:22
  std::vector<double> tab((size_t)f.m * 2 * n);
  for (int t = 0; t < f.m; ++t)
    for (int c = 0; c < n; ++c)
      for (int b = 0; b < 2; ++b)  // point coordinate (c + offset) * h, fem.hpp:155-157
        tab[(size_t)t * 2 * n + 2 * c + b] = kl_axis_eval(f, t, (c + off[b]) * h);
  return tab;
}

void make_asm_tables(AsmTables& T, int n, double alpha, double beta, const double velocity[3]) {
  // BasisTables (fem.hpp:81-97)
  double value[8][8], gradient[8][8][3];
  const double g = 1.0 / std::sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
    for (int c = 0; c < 8; ++c) {
      const double sg[3] = {(c & 1) ? 1.0 : -1.0, (c & 2) ? 1.0 : -1.0, (c & 4) ? 1.0 : -1.0};
      const double lin[3] = {0.5 * (1.0 + sg[0] * xi[0]), 0.5 * (1.0 + sg[1] * xi[1]),
                             0.5 * (1.0 + sg[2] * xi[2])};
      value[q][c] = lin[0] * lin[1] * lin[2];
      gradient[q][c][0] = 0.5 * sg[0] * lin[1] * lin[2];
      gradient[q][c][1] = lin[0] * 0.5 * sg[1] * lin[2];
      gradient[q][c][2] = lin[0] * lin[1] * 0.5 * sg[2];
    }
  }
  const double h = 1.0 / n;
  const double grad_scale = 2.0 / h;                                    // fem.hpp:135
  T.wd = (h / 2.0) * (h / 2.0) * (h / 2.0);                              // fem.hpp:136
  const double vx = velocity[0], vy = velocity[1], vz = velocity[2];
  T.alpha = alpha;
  T.beta = beta;
  T.vx = vx;
  T.vy = vy;
  T.vz = vz;
  for (int q = 0; q < 8; ++q) {
    for (int c = 0; c < 8; ++c) {
      T.VAL[q][c] = value[q][c];
      for (int a = 0; a < 3; ++a) T.GS[q][c][a] = gradient[q][c][a] * grad_scale;  // fem.hpp:163-165
    }
    for (int i = 0; i < 8; ++i) {
      const double gx_i = gradient[q][i][0] * grad_scale;  // fem.hpp:172-175
      const double gy_i = gradient[q][i][1] * grad_scale;
      const double gz_i = gradient[q][i][2] * grad_scale;
      const double n_i = value[q][i];
      for (int j = 0; j < 8; ++j) {
        const double gx_j = gradient[q][j][0] * grad_scale;  // fem.hpp:183-186
        const double gy_j = gradient[q][j][1] * grad_scale;
        const double gz_j = gradient[q][j][2] * grad_scale;
        const double n_j = value[q][j];
        T.ADV[q][i][j] = alpha * (vx * gx_j + vy * gy_j + vz * gz_j) * n_i;  // fem.hpp:187
        T.G[q][i][j] = gx_j * gx_i + gy_j * gy_i + gz_j * gz_i;               // fem.hpp:190
        T.NN[q][i][j] = n_j * n_i;                                            // fem.hpp:191
      }
    }
  }
}

}  // namespace ep
