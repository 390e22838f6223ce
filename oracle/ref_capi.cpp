// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" shim over the *unmodified* reference library
// (/root/reference/proj), compiled by oracle/Makefile into
// oracle/_ref/libenprop_ref.so. Every function below forwards to the
// reference's own templates so that tests and bench.py's reference arm can
// run the reference algorithm on plain arrays:
//   build_node_graph      proj/src/mesh.cpp:13-55
//   KlField               proj/include/enprop/kl.hpp:39-95, proj/src/kl.cpp:64-89
//   assemble              proj/include/enprop/fem.hpp:115-202
//   apply_dirichlet       proj/include/enprop/fem.hpp:218-243
//   spmv / dot / axpby    proj/include/enprop/kernels.hpp:15-85
//   pcg_solve             proj/include/enprop/pcg.hpp:52-103
//   draw_samples          proj/src/samples.cpp:7-18
//   partition / distributed_spmv   proj/src/partition.cpp:31-72, proj/include/enprop/halo.hpp:169-202
//
// Array layouts are the reference's own memory layouts: Ensemble<S> is a POD
// of S doubles (ensemble.hpp:105-106), so CrsMatrix<Ensemble<S>>::values is
// [nnz][S] and DenseVector<Ensemble<S>> is [rows][S].
#include <algorithm>
#include <chrono>
#include <random>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "enprop/ensemble.hpp"
#include "enprop/crs.hpp"
#include "enprop/kernels.hpp"
#include "enprop/kl.hpp"
#include "enprop/mesh.hpp"
#include "enprop/fem.hpp"
#include "enprop/pcg.hpp"
#include "enprop/samples.hpp"
#include "enprop/partition.hpp"
#include "enprop/halo.hpp"
#include "enprop/multigrid.hpp"

using namespace enprop;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SolverError& e) {
    g_err = e.what();
    return std::string(e.what()).find("positive definite") != std::string::npos ? 3 : 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename F>
void with_width(int s, F&& f) {
  switch (s) {
    case 1: f(std::integral_constant<int, 1>()); return;
    case 2: f(std::integral_constant<int, 2>()); return;
    case 4: f(std::integral_constant<int, 4>()); return;
    case 8: f(std::integral_constant<int, 8>()); return;
    case 16: f(std::integral_constant<int, 16>()); return;
    case 32: f(std::integral_constant<int, 32>()); return;
    default: throw std::invalid_argument("ensemble width outside {1,2,4,8,16,32}");
  }
}

// Scalar type for width S: plain double at S=1 when `scalar` is requested
// (the reference's own per-sample path), else Ensemble<S>.
template <int S>
using E = Ensemble<S>;

template <typename T>
std::vector<T> from_raw(const double* p, std::size_t n) {
  std::vector<T> v(n);
  std::memcpy(static_cast<void*>(v.data()), p, n * sizeof(T));
  return v;
}

template <typename T>
void to_raw(const std::vector<T>& v, double* p) {
  std::memcpy(p, static_cast<const void*>(v.data()), v.size() * sizeof(T));
}

template <typename T>
CrsMatrix<T> make_matrix(int rows, int cols, const int* row_map, const int* col_entry,
                         const double* values) {
  CrsMatrix<T> a;
  a.num_rows = rows;
  a.num_cols = cols;
  a.row_map.assign(row_map, row_map + rows + 1);
  const int nnz = row_map[rows];
  a.col_entry.assign(col_entry, col_entry + nnz);
  a.values = from_raw<T>(values, nnz);
  return a;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int64_t ref_graph_nnz(int n) {
  const int64_t npa = n + 1;
  const int64_t t = 3 * npa - 2;
  return t * t * t;
}

int ref_build_graph(int n, int* row_map, int* col_entry) {
  return guarded([&] {
    StructuredMesh mesh(n);
    Graph g = build_node_graph(mesh);
    std::memcpy(row_map, g.row_map.data(), g.row_map.size() * sizeof(int));
    std::memcpy(col_entry, g.col_entry.data(), g.col_entry.size() * sizeof(int));
  });
}

// entry_of_pair table of AssemblyContext (fem.hpp:45-56): cells*64 ints.
int ref_entry_of_pair(int n, int* out) {
  return guarded([&] {
    StructuredMesh mesh(n);
    AssemblyContext ctx(mesh);
    for (int cell = 0; cell < mesh.num_cells(); ++cell)
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) out[(std::size_t)cell * 64 + i * 8 + j] = ctx.entry_of_pair(cell, i, j);
  });
}

// KL field description: per retained mode i: axis triple + eigenvalue; per
// axis mode t: frequency, eigenvalue, inverse_norm, cosine flag.
int ref_kl_describe(int m, double mean, double sigma, double L, int* mode_axes /*m*3*/,
                    double* mode_eig /*m*/, double* axis_freq /*m*/, double* axis_eig /*m*/,
                    double* axis_invnorm /*m*/, int* axis_cos /*m*/) {
  return guarded([&] {
    KlField f(m, mean, sigma, L);
    for (int i = 0; i < m; ++i) {
      auto ax = f.axis_modes(i);
      for (int a = 0; a < 3; ++a) mode_axes[i * 3 + a] = ax[a];
      mode_eig[i] = f.eigenvalue(i);
    }
    const auto& am = f.axis_eigenpairs();
    for (int t = 0; t < (int)am.size(); ++t) {
      axis_freq[t] = am[t].frequency;
      axis_eig[t] = am[t].eigenvalue;
      axis_invnorm[t] = am[t].inverse_norm;
      axis_cos[t] = am[t].cosine_branch ? 1 : 0;
    }
  });
}

// KlField::evaluate<Ensemble<S>> at one point (kl.hpp:67-81). y is [m][S].
int ref_kl_evaluate(int s, int m, double mean, double sigma, double L, const double* x3,
                    const double* y, double* out) {
  return guarded([&] {
    KlField f(m, mean, sigma, L);
    std::array<double, 3> x = {x3[0], x3[1], x3[2]};
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      auto yy = from_raw<E<S>>(y, m);
      E<S> k = f.evaluate<E<S>>(x, std::span<const E<S>>(yy));
      std::memcpy(out, k.data(), sizeof(double) * S);
    });
  });
}

// assemble<Ensemble<S>> (+ optional apply_dirichlet). u: [rows][S] (nullptr = 0);
// y: [m][S]; values: [nnz][S]; residual: [rows][S].
// scalar != 0 with s == 1 runs the reference's assemble<double> path instead.
int ref_assemble(int s, int scalar, int n, int m, double mean, double sigma, double L,
                 double alpha, double beta, const double* velocity, const double* u,
                 const double* y, int dirichlet, double bc_x0, double bc_x1, double* values,
                 double* residual) {
  return guarded([&] {
    StructuredMesh mesh(n);
    AssemblyContext ctx(mesh);
    KlField field(m, mean, sigma, L);
    PdeCoefficients coeffs;
    coeffs.alpha = alpha;
    coeffs.beta = beta;
    if (velocity) coeffs.velocity = {velocity[0], velocity[1], velocity[2]};
    DirichletBc bc{bc_x0, bc_x1};
    const std::size_t rows = mesh.num_nodes();
    auto run = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> uu(rows, T(0.0));
      if (u) uu = from_raw<T>(u, rows);
      auto yy = from_raw<T>(y, m);
      AssembledSystem<T> sys;
      assemble<T>(ctx, field, coeffs, uu, std::span<const T>(yy), sys);
      if (dirichlet) apply_dirichlet(sys, mesh, bc, uu);
      to_raw(sys.matrix.values, values);
      to_raw(sys.residual, residual);
    };
    if (scalar && s == 1) {
      run(double{});
    } else {
      with_width(s, [&](auto w) { run(E<decltype(w)::value>{}); });
    }
  });
}

// apply_dirichlet alone on given values/residual (in place).
int ref_apply_dirichlet(int s, int n, double bc_x0, double bc_x1, const double* u,
                        double* values, double* residual) {
  return guarded([&] {
    StructuredMesh mesh(n);
    Graph g = build_node_graph(mesh);
    DirichletBc bc{bc_x0, bc_x1};
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      AssembledSystem<E<S>> sys;
      sys.matrix = make_matrix<E<S>>(g.num_rows, g.num_cols, g.row_map.data(), g.col_entry.data(), values);
      sys.residual = from_raw<E<S>>(residual, g.num_rows);
      std::vector<E<S>> uu(g.num_rows, E<S>(0.0));
      if (u) uu = from_raw<E<S>>(u, g.num_rows);
      apply_dirichlet(sys, mesh, bc, uu);
      to_raw(sys.matrix.values, values);
      to_raw(sys.residual, residual);
    });
  });
}

int ref_spmv(int s, int rows, int cols, const int* row_map, const int* col_entry,
             const double* values, const double* x, double* z) {
  return guarded([&] {
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      auto a = make_matrix<E<S>>(rows, cols, row_map, col_entry, values);
      auto xx = from_raw<E<S>>(x, cols);
      std::vector<E<S>> zz;
      spmv(a, xx, zz);
      to_raw(zz, z);
    });
  });
}

// spmv_outer on OuterEnsembleMatrix (kernels.hpp:38-56, crs.hpp:138-147).
int ref_spmv_outer(int s, int rows, int cols, const int* row_map, const int* col_entry,
                   const double* values, const double* x, double* z) {
  return guarded([&] {
    OuterEnsembleMatrix a;
    a.num_rows = rows;
    a.num_cols = cols;
    a.ensemble_size = s;
    a.row_map.assign(row_map, row_map + rows + 1);
    a.col_entry.assign(col_entry, col_entry + row_map[rows]);
    a.values.assign(values, values + (size_t)row_map[rows] * s);
    DenseVector<double> xx(x, x + (size_t)cols * s), zz;
    spmv_outer(a, xx, zz);
    std::copy(zz.begin(), zz.end(), z);
  });
}

// Coupled dot (kernels.hpp:62-69).
int ref_dot(int s, int64_t n, const double* u, const double* v, double* out) {
  return guarded([&] {
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      auto uu = from_raw<E<S>>(u, n);
      auto vv = from_raw<E<S>>(v, n);
      *out = dot(uu, vv);
    });
  });
}

// axpby (kernels.hpp:78-85); per_lane selects Ensemble coefficients.
int ref_axpby(int s, int64_t n, int per_lane, const double* alpha, const double* x,
              const double* beta, double* y) {
  return guarded([&] {
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      auto xx = from_raw<E<S>>(x, n);
      auto yy = from_raw<E<S>>(y, n);
      if (per_lane) {
        E<S> a, b;
        for (int e = 0; e < S; ++e) { a[e] = alpha[e]; b[e] = beta[e]; }
        axpby(a, xx, b, yy);
      } else {
        axpby(alpha[0], xx, beta[0], yy);
      }
      to_raw(yy, y);
    });
  });
}

// pcg_solve<Ensemble<S>>(IdentityPreconditioner) (pcg.hpp:52-103), or
// pcg_solve<double> when scalar && s == 1. history must hold maxit+1 doubles.
// Returns 0 ok, 2 no convergence, 3 indefinite, 1 invalid.
int ref_pcg(int s, int scalar, int rows, const int* row_map, const int* col_entry,
            const double* values, const double* b, double tol, int maxit, double* x,
            int* iterations, double* history, int* hist_len) {
  *hist_len = 0;
  *iterations = -1;
  return guarded([&] {
    SolverConfig cfg;
    cfg.tol = tol;
    cfg.max_iterations = maxit;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      auto a = make_matrix<T>(rows, rows, row_map, col_entry, values);
      auto bb = from_raw<T>(b, rows);
      try {
        auto res = pcg_solve(a, bb, IdentityPreconditioner{}, cfg);
        to_raw(res.solution, x);
        *iterations = res.iterations;
        for (std::size_t i = 0; i < res.residual_history.size(); ++i) history[i] = res.residual_history[i];
        *hist_len = (int)res.residual_history.size();
      } catch (const SolverError& err) {
        for (std::size_t i = 0; i < err.history().size(); ++i) history[i] = err.history()[i];
        *hist_len = (int)err.history().size();
        throw;
      }
    };
    if (scalar && s == 1) run(double{});
    else with_width(s, [&](auto w) { run(E<decltype(w)::value>{}); });
  });
}

// newton_solve (fem.hpp:265-302) composed from the reference's own pieces with
// the multigrid preconditioner replaced by IdentityPreconditioner (the loop
// below is fem.hpp:273-301 line for line otherwise): coupled ensemble CG.
int ref_newton_identity(int s, int scalar, int n, int m, double mean, double sigma, double L,
                        double alpha, double beta, const double* velocity, const double* y,
                        double bc_x0, double bc_x1, double tol, int max_newton, double lin_tol,
                        int lin_maxit, double* u_out, int* iterations, int* total_cg,
                        double* norms, int* num_norms) {
  *iterations = 0;
  *total_cg = 0;
  *num_norms = 0;
  return guarded([&] {
    StructuredMesh mesh(n);
    AssemblyContext ctx(mesh);
    KlField field(m, mean, sigma, L);
    PdeCoefficients coeffs;
    coeffs.alpha = alpha;
    coeffs.beta = beta;
    if (velocity) coeffs.velocity = {velocity[0], velocity[1], velocity[2]};
    DirichletBc bc{bc_x0, bc_x1};
    SolverConfig linear;
    linear.tol = lin_tol;
    linear.max_iterations = lin_maxit;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      auto yy = from_raw<T>(y, m);
      DenseVector<T> sol(mesh.num_nodes(), T(0.0));
      AssembledSystem<T> system;
      double initial_norm = 0.0;
      auto out = [&] {
        to_raw(sol, u_out);
      };
      for (int step = 0;; ++step) {
        assemble<T>(ctx, field, coeffs, sol, std::span<const T>(yy), system);
        apply_dirichlet(system, mesh, bc, sol);
        const double residual_norm = norm2(system.residual);
        norms[(*num_norms)++] = residual_norm;
        if (step == 0) {
          initial_norm = residual_norm;
          if (initial_norm == 0.0) return out();
        } else if (residual_norm < tol * initial_norm) {
          *iterations = step;
          return out();
        }
        if (step >= max_newton) {
          *iterations = step;
          out();
          throw SolverError("newton_solve: no convergence", {});
        }
        DenseVector<T> rhs(system.residual.size());
        for (std::size_t i = 0; i < rhs.size(); ++i) rhs[i] = -system.residual[i];
        SolveResult<T> lin = pcg_solve(system.matrix, rhs, IdentityPreconditioner{}, linear);
        *total_cg += lin.iterations;
        axpby(1.0, lin.solution, 1.0, sol);
      }
    };
    if (scalar && s == 1) run(double{});
    else with_width(s, [&](auto w) { run(E<decltype(w)::value>{}); });
  });
}

// write_exchange_trace_csv (halo.cpp:192-202) on given records
int ref_write_trace_csv(const char* path, int n, const int* rank, const int* nb, const int64_t* bytes,
                        const double* t) {
  return guarded([&] {
    std::vector<ExchangeRecord> tr(n);
    for (int i = 0; i < n; ++i) tr[i] = ExchangeRecord{rank[i], nb[i], bytes[i], t[i]};
    write_exchange_trace_csv(path, tr);
  });
}

// fit_halo_model / predicted_speedup (halo.cpp:156-188).
int ref_fit_halo_model(int n, const double* s, const double* t, double* a, double* b, double* rss) {
  return guarded([&] {
    std::vector<std::pair<double, double>> samples;
    for (int i = 0; i < n; ++i) samples.emplace_back(s[i], t[i]);
    const HaloFit fit = fit_halo_model(samples);
    *a = fit.model.a;
    *b = fit.model.b;
    *rss = fit.residual_sum_of_squares;
  });
}

int ref_predicted_speedup(double a, double b, double s, double* out) {
  return guarded([&] {
    HaloModel m;
    m.a = a;
    m.b = b;
    *out = predicted_speedup(m, s);
  });
}

// draw_samples(seed, count, m) (samples.cpp:7-18) -> out[count][m].
int ref_draw_samples(uint64_t seed, int count, int m, double* out) {
  return guarded([&] {
    auto v = draw_samples(seed, count, m);
    for (int i = 0; i < count; ++i)
      for (int j = 0; j < m; ++j) out[(std::size_t)i * m + j] = v[i][j];
  });
}

// Slab partition (partition.cpp:31-72): ranges[p][2] = {first_plane, num_planes}.
int ref_partition(int n, int p, int* ranges) {
  return guarded([&] {
    StructuredMesh mesh(n);
    auto part = partition(mesh, p);
    for (int r = 0; r < p; ++r) {
      ranges[2 * r] = part.ranges[r].first_plane;
      ranges[2 * r + 1] = part.ranges[r].num_planes;
    }
  });
}

// distributed_spmv over the reference's x-slab partition (halo.hpp:169-202).
int ref_distributed_spmv(int s, int n, int p, const double* values, const double* x, double* z,
                         int* num_messages) {
  return guarded([&] {
    StructuredMesh mesh(n);
    Graph g = build_node_graph(mesh);
    auto part = partition(mesh, p);
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      auto a = make_matrix<E<S>>(g.num_rows, g.num_cols, g.row_map.data(), g.col_entry.data(), values);
      auto xx = from_raw<E<S>>(x, g.num_rows);
      auto res = distributed_spmv(part, a, xx, TransportModel{});
      to_raw(res.product, z);
      *num_messages = res.exchange.num_messages;
    });
  });
}

// ---------------------------------------------------------------------------
// Timed CPU baseline (bench.py --impl reference): one ensemble group of width
// S through the reference's own path — pack_sample_group, assemble,
// apply_dirichlet, rhs = -residual (bench.cpp:294-299), then pcg_solve with
// IdentityPreconditioner. coupled=1 runs pcg_solve<Ensemble<S>>; coupled=0
// runs S x (extract_component + pcg_solve<double>) (bench.cpp:340-349).
// max_cg caps the iterations actually run (a bounded sample); the call then
// reports per-iteration time so the caller can scale by a full solve's count.
// times[0]=assembly+dirichlet s, times[1]=cg s, times[2]=cg iterations run.
// times[0] assembly + Dirichlet, [1] CG (incl. extraction), [2] CG iterations
// run, [3] extract_component time (uncoupled only; 0 otherwise)
int ref_time_group(int s, int coupled, int n, int m, double mean, double sigma, double L,
                   uint64_t seed, int group, double tol, int max_cg, double* times,
                   int* iterations /*S*/) {
  return guarded([&] {
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      using T = E<S>;
      using clock = std::chrono::steady_clock;
      StructuredMesh mesh(n);
      AssemblyContext ctx(mesh);
      KlField field(m, mean, sigma, L);
      auto pool = draw_samples(seed, (group + 1) * S, m);
      auto y = pack_sample_group<S>(pool, group * S);
      const int nodes = mesh.num_nodes();
      auto t0 = clock::now();
      DenseVector<T> u0(nodes, T(0.0));
      AssembledSystem<T> sys;
      assemble(ctx, field, PdeCoefficients{}, u0, std::span<const T>(y), sys);
      apply_dirichlet(sys, mesh, DirichletBc{}, u0);
      DenseVector<T> rhs(nodes);
      for (int i = 0; i < nodes; ++i) rhs[i] = -sys.residual[i];
      auto t1 = clock::now();
      SolverConfig cfg;
      cfg.tol = tol;
      cfg.max_iterations = max_cg;
      int ran = 0;
      if (coupled) {
        try {
          auto r = pcg_solve(sys.matrix, rhs, IdentityPreconditioner{}, cfg);
          for (int e = 0; e < S; ++e) iterations[e] = r.iterations;
          ran = r.iterations;
        } catch (const SolverError& err) {
          for (int e = 0; e < S; ++e) iterations[e] = -1;
          ran = (int)err.history().size() - 1;
        }
      } else {
        CrsMatrix<double> ae;
        DenseVector<double> be;
        double t_extract = 0.0;
        for (int e = 0; e < S; ++e) {
          auto te = clock::now();
          extract_component(sys.matrix, e, ae);
          extract_component(rhs, e, be);
          t_extract += std::chrono::duration<double>(clock::now() - te).count();
          try {
            auto r = pcg_solve(ae, be, IdentityPreconditioner{}, cfg);
            iterations[e] = r.iterations;
            ran += r.iterations;
          } catch (const SolverError& err) {
            iterations[e] = -1;
            ran += (int)err.history().size() - 1;
          }
        }
        times[3] = t_extract;
      }
      auto t2 = clock::now();
      times[0] = std::chrono::duration<double>(t1 - t0).count();
      times[1] = std::chrono::duration<double>(t2 - t1).count();
      times[2] = ran;
    });
  });
}

// ---- multigrid (multigrid.hpp): the reference's own hierarchy, V-cycle and
// MG-preconditioned pcg_solve, for the f4 parity tests. `scalar` with s == 1
// uses the plain-double hierarchy (the per-sample path of bench.cpp:322-330).
}  // extern "C"

static MgOptions mg_options(int thr, int deg, double ratio, double boost, int pits) {
  MgOptions o;
  o.coarse_row_threshold = thr;
  o.chebyshev_degree = deg;
  o.eigenvalue_ratio = ratio;
  o.eigenvalue_boost = boost;
  o.power_iterations = pits;
  return o;
}

template <typename F>
static void with_scalar(int s, int scalar, F&& f) {
  if (scalar && s == 1) f(double{});
  else with_width(s, [&](auto w) { f(E<decltype(w)::value>{}); });
}

extern "C" {

// levels, rows per level, lambda_max [levels-1][s]
int ref_mg_describe(int s, int scalar, int rows, const int* row_map, const int* col_entry, const double* values,
                    int thr, int deg, double ratio, double boost, int pits, int* num_levels, int* level_rows,
                    int max_levels, double* lambda_max) {
  return guarded([&] {
    with_scalar(s, scalar, [&](auto tag) {
      using T = decltype(tag);
      auto a = make_matrix<T>(rows, rows, row_map, col_entry, values);
      MgHierarchy<T> h = build_hierarchy(a, mg_options(thr, deg, ratio, boost, pits));
      *num_levels = h.num_levels();
      for (int k = 0; k < h.num_levels() && k < max_levels; ++k) {
        level_rows[k] = h.levels[k].a.num_rows;
        if (k + 1 < h.num_levels()) {
          const T lm = h.levels[k].smoother.lambda_max;
          std::memcpy(lambda_max + (size_t)k * s, &lm, sizeof(T));
        }
      }
    });
  });
}

// one V-cycle on level 0: x updated in place
int ref_mg_vcycle(int s, int scalar, int rows, const int* row_map, const int* col_entry, const double* values,
                  int thr, int deg, double ratio, double boost, int pits, const double* b, double* x) {
  return guarded([&] {
    with_scalar(s, scalar, [&](auto tag) {
      using T = decltype(tag);
      auto a = make_matrix<T>(rows, rows, row_map, col_entry, values);
      MgHierarchy<T> h = build_hierarchy(a, mg_options(thr, deg, ratio, boost, pits));
      auto bb = from_raw<T>(b, rows);
      auto xx = from_raw<T>(x, rows);
      vcycle(h, bb, xx);
      to_raw(xx, x);
    });
  });
}

// pcg_solve(a, b, MgPreconditioner(h), cfg); history must hold maxit+1 doubles
int ref_mg_pcg(int s, int scalar, int rows, const int* row_map, const int* col_entry, const double* values,
               int thr, int deg, double ratio, double boost, int pits, const double* b, double tol, int maxit,
               double* x, int* iterations, double* history, int* hist_len) {
  *hist_len = 0;
  *iterations = -1;
  return guarded([&] {
    with_scalar(s, scalar, [&](auto tag) {
      using T = decltype(tag);
      auto a = make_matrix<T>(rows, rows, row_map, col_entry, values);
      MgHierarchy<T> h = build_hierarchy(a, mg_options(thr, deg, ratio, boost, pits));
      auto bb = from_raw<T>(b, rows);
      SolverConfig cfg;
      cfg.tol = tol;
      cfg.max_iterations = maxit;
      try {
        auto res = pcg_solve(a, bb, MgPreconditioner<T>(h), cfg);
        to_raw(res.solution, x);
        *iterations = res.iterations;
        for (std::size_t i = 0; i < res.residual_history.size(); ++i) history[i] = res.residual_history[i];
        *hist_len = (int)res.residual_history.size();
      } catch (const SolverError& err) {
        for (std::size_t i = 0; i < err.history().size(); ++i) history[i] = err.history()[i];
        *hist_len = (int)err.history().size();
        throw;
      }
    });
  });
}

// the reference's own newton_solve (fem.hpp:265-302): multigrid-preconditioned
// coupled linear solves, default MgOptions unless given
int ref_newton_mg(int s, int scalar, int n, int m, double mean, double sigma, double L, double alpha,
                  double beta, const double* velocity, const double* y, double bc_x0, double bc_x1, double tol,
                  int max_newton, double lin_tol, int lin_maxit, int thr, int deg, double ratio, double boost,
                  int pits, double* u_out, int* iterations, int* total_cg, double* norms, int* num_norms) {
  *iterations = 0;
  *total_cg = 0;
  *num_norms = 0;
  return guarded([&] {
    StructuredMesh mesh(n);
    KlField field(m, mean, sigma, L);
    PdeCoefficients coeffs;
    coeffs.alpha = alpha;
    coeffs.beta = beta;
    if (velocity) coeffs.velocity = {velocity[0], velocity[1], velocity[2]};
    NewtonOptions opt;
    opt.tol = tol;
    opt.max_iterations = max_newton;
    opt.linear.tol = lin_tol;
    opt.linear.max_iterations = lin_maxit;
    opt.multigrid = mg_options(thr, deg, ratio, boost, pits);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      auto yy = from_raw<T>(y, m);
      try {
        NewtonResult<T> r = newton_solve<T>(mesh, field, coeffs, yy, DirichletBc{bc_x0, bc_x1}, opt);
        to_raw(r.solution, u_out);
        *iterations = r.iterations;
        *total_cg = r.total_cg_iterations;
        for (double v : r.residual_norms) norms[(*num_norms)++] = v;
      } catch (const SolverError& err) {
        for (double v : err.history()) norms[(*num_norms)++] = v;
        throw;
      }
    };
    if (scalar && s == 1) run(double{});
    else with_width(s, [&](auto w) { run(E<decltype(w)::value>{}); });
  });
}

// Timed reference spmv<Ensemble<S>> on the assembled+Dirichlet matrix, best of reps.
int ref_time_spmv(int s, int n, int m, double mean, double sigma, double L, uint64_t seed,
                  int reps, double* best_seconds) {
  return guarded([&] {
    with_width(s, [&](auto w) {
      constexpr int S = decltype(w)::value;
      using T = E<S>;
      StructuredMesh mesh(n);
      AssemblyContext ctx(mesh);
      KlField field(m, mean, sigma, L);
      auto pool = draw_samples(seed, S, m);
      auto y = pack_sample_group<S>(pool, 0);
      DenseVector<T> u0(mesh.num_nodes(), T(0.0));
      AssembledSystem<T> sys;
      assemble(ctx, field, PdeCoefficients{}, u0, std::span<const T>(y), sys);
      apply_dirichlet(sys, mesh, DirichletBc{}, u0);
      std::mt19937_64 rng(seed + 0x9e3779b97f4a7c15ull);
      DenseVector<T> x(sys.matrix.num_cols);
      for (auto& v : x)
        for (int e = 0; e < S; ++e) v[e] = double(rng() >> 11) * (2.0 / 9007199254740992.0) - 1.0;
      DenseVector<T> z;
      double best = 1e300;
      for (int r = 0; r < reps; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        spmv(sys.matrix, x, z);
        auto t1 = std::chrono::steady_clock::now();
        best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
      }
      *best_seconds = best;
    });
  });
}

}  // extern "C"
