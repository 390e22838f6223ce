// Drop-in test: the reference's own C++ types and call sites, with the
// namespace switched to enprop_b200, must give the reference's results bit for
// bit. Mirrors proj/tests/test_kernels.cpp (ensemble SpMV, coupled dot,
// axpby), test_mesh_fem.cpp (graph, ensemble assembly, Dirichlet) and
// test_pcg.cpp (coupled CG, iteration exhaustion with history).
//
// Built by tests/cpp/Makefile where /root/reference exists (compile time only);
// the binary runs on the GPU box from tests/test_cpp_dropin.py.
#include <cstdio>
#include <cstring>
#include <random>
#include <span>
#include <vector>

#include "enprop/crs.hpp"
#include "enprop/ensemble.hpp"
#include "enprop/fem.hpp"
#include "enprop/kernels.hpp"
#include "enprop/kl.hpp"
#include "enprop/mesh.hpp"
#include "enprop/pcg.hpp"
#include "enprop/samples.hpp"
#include "oracles.hpp"  // proj/tests/oracles.hpp: random_crs, uniform_pm1

#define ENPROP_B200_SOLVER_ERROR ::enprop::SolverError
#include "enprop_b200/dropin.hpp"

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                    \
  } while (0)

template <class T>
static bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0;
}

using namespace enprop;
static std::mt19937_64 rng(771420u);

template <int S>
static void spmv_dot_axpby() {
  for (int trial = 0; trial < 10; ++trial) {
    const int rows = 1 + static_cast<int>(rng() % 60), cols = 1 + static_cast<int>(rng() % 60);
    CrsMatrix<double> base = testutil::random_crs(rng, rows, cols, 0.15);
    std::vector<CrsMatrix<double>> parts(S, base);
    for (auto& p : parts)
      for (auto& v : p.values) v = testutil::uniform_pm1(rng);
    auto a = pack_matrix<S>(parts);
    DenseVector<Ensemble<S>> x(cols);
    for (auto& v : x)
      for (int e = 0; e < S; ++e) v[e] = testutil::uniform_pm1(rng);
    CHECK(same_bits(enprop::spmv(a, x), enprop_b200::spmv(a, x)));
  }
  DenseVector<Ensemble<S>> u(777), v(777);
  for (auto* w : {&u, &v})
    for (auto& r : *w)
      for (int e = 0; e < S; ++e) r[e] = testutil::uniform_pm1(rng);
  CHECK(enprop::dot(u, v) == enprop_b200::dot(u, v));
  CHECK(enprop::norm2(u) == enprop_b200::norm2(u));
  auto y1 = v, y2 = v;
  enprop::axpby(2.5, u, -0.75, y1);
  enprop_b200::axpby(2.5, u, -0.75, y2);
  CHECK(same_bits(y1, y2));
  Ensemble<S> al, be;
  for (int e = 0; e < S; ++e) {
    al[e] = testutil::uniform_pm1(rng);
    be[e] = testutil::uniform_pm1(rng);
  }
  y1 = v;
  y2 = v;
  enprop::axpby(al, u, be, y1);
  enprop_b200::axpby(al, u, be, y2);
  CHECK(same_bits(y1, y2));
}

// sample-major layout (test_kernels.cpp:127-143): spmv_outer on OuterEnsembleMatrix
static void spmv_outer_layout(int s) {
  for (int trial = 0; trial < 10; ++trial) {
    const int rows = 1 + static_cast<int>(rng() % 60), cols = 1 + static_cast<int>(rng() % 60);
    CrsMatrix<double> base = testutil::random_crs(rng, rows, cols, 0.15);
    OuterEnsembleMatrix a;
    a.num_rows = rows;
    a.num_cols = cols;
    a.ensemble_size = s;
    a.row_map = base.row_map;
    a.col_entry = base.col_entry;
    a.values.resize(base.col_entry.size() * s);
    for (auto& v : a.values) v = testutil::uniform_pm1(rng);
    DenseVector<double> x(static_cast<std::size_t>(cols) * s), z1, z2;
    for (auto& v : x) v = testutil::uniform_pm1(rng);
    enprop::spmv_outer(a, x, z1);
    enprop_b200::spmv_outer(a, x, z2);
    CHECK(same_bits(z1, z2));
  }
}

template <class Scalar>
static void assembly_and_cg(int n) {
  StructuredMesh mesh(n);
  AssemblyContext ctx(mesh);
  KlField field(5, 1.0, 0.2, 1.0);
  constexpr int S = sizeof(Scalar) / sizeof(double);
  auto pool = draw_samples(515, S, 5);
  std::vector<Scalar> y(5);
  for (int j = 0; j < 5; ++j)
    for (int e = 0; e < S; ++e) reinterpret_cast<double*>(&y[j])[e] = pool[e][j];
  std::vector<Scalar> u(mesh.num_nodes());
  for (auto& v : u)
    for (int e = 0; e < S; ++e) reinterpret_cast<double*>(&v)[e] = testutil::uniform_pm1(rng);
  const PdeCoefficients nonlinear{0.3, 0.7, {1.0, 0.5, -0.25}};
  AssembledSystem<Scalar> ref, ours;
  enprop::assemble<Scalar>(ctx, field, nonlinear, u, std::span<const Scalar>(y), ref);
  enprop_b200::assemble(ctx, field, nonlinear, u, std::span<const Scalar>(y), ours);
  CHECK(ref.matrix.row_map == ours.matrix.row_map);
  CHECK(ref.matrix.col_entry == ours.matrix.col_entry);
  CHECK(same_bits(ref.matrix.values, ours.matrix.values));
  CHECK(same_bits(ref.residual, ours.residual));
  enprop::apply_dirichlet(ref, mesh, DirichletBc{}, u);
  enprop_b200::apply_dirichlet(ours, mesh, DirichletBc{}, u);
  CHECK(same_bits(ref.matrix.values, ours.matrix.values));
  CHECK(same_bits(ref.residual, ours.residual));

  // the linear bench problem (bench.cpp:294-299): u = 0, rhs = -residual
  std::vector<Scalar> u0(mesh.num_nodes(), Scalar(0.0));
  enprop::assemble<Scalar>(ctx, field, PdeCoefficients{}, u0, std::span<const Scalar>(y), ref);
  enprop::apply_dirichlet(ref, mesh, DirichletBc{}, u0);
  std::vector<Scalar> b(ref.residual.size());
  for (size_t i = 0; i < b.size(); ++i) b[i] = -ref.residual[i];
  SolverConfig cfg;
  cfg.tol = 1e-8;
  auto r1 = enprop::pcg_solve(ref.matrix, b, IdentityPreconditioner{}, cfg);
  auto r2 = enprop_b200::pcg_solve(ref.matrix, b, IdentityPreconditioner{}, cfg);
  CHECK(r1.iterations == r2.iterations);
  CHECK(same_bits(r1.solution, r2.solution));
  CHECK(same_bits(r1.residual_history, r2.residual_history));
}

template <int S>
static void uncoupled_is_per_sample_scalar(int n) {
  StructuredMesh mesh(n);
  AssemblyContext ctx(mesh);
  KlField field(10, 1.0, 0.25, 1.0);
  auto y = pack_sample_group<S>(draw_samples(4, S, 10), 0);
  DenseVector<Ensemble<S>> u0(mesh.num_nodes(), Ensemble<S>(0.0));
  auto sys = enprop::assemble<Ensemble<S>>(ctx, field, PdeCoefficients{}, u0, std::span<const Ensemble<S>>(y));
  enprop::apply_dirichlet(sys, mesh, DirichletBc{}, u0);
  DenseVector<Ensemble<S>> b(sys.residual.size());
  for (size_t i = 0; i < b.size(); ++i) b[i] = -sys.residual[i];
  SolverConfig cfg;
  cfg.tol = 1e-6;
  auto ens = enprop_b200::pcg_solve_uncoupled(sys.matrix, b, cfg);
  for (int e = 0; e < S; ++e) {
    auto ae = extract_component(sys.matrix, e);
    auto be = extract_component(b, e);
    auto ref = enprop::pcg_solve(ae, be, IdentityPreconditioner{}, cfg);
    CHECK(ens.iterations[e] == ref.iterations);
    CHECK(ens.status[e] == 0);
    bool same = true;
    for (size_t i = 0; i < be.size(); ++i)
      same &= std::memcmp(&ens.solution[i][e], &ref.solution[i], sizeof(double)) == 0;
    CHECK(same);
    CHECK(ens.residual_history[e] == ref.residual_history);
  }
}

// value-returning assemble (fem.hpp:204-210), the reference's result types
// through the drop-in, and draw_samples / pack_sample_group (samples.cpp:7-18)
template <int S>
static void value_forms_and_samples(int n) {
  StructuredMesh mesh(n);
  AssemblyContext ctx(mesh);
  KlField field(3, 1.0, 0.1, 1.0);
  const auto pool = draw_samples(0, 3 * S, 3);
  const auto pool2 = enprop_b200::draw_samples(0, 3 * S, 3);
  CHECK(pool == pool2);
  const auto y = pack_sample_group<S>(pool, S);
  const auto y2 = enprop_b200::pack_sample_group<Ensemble<S>>(pool2, S);
  CHECK(same_bits(y, y2));
  DenseVector<Ensemble<S>> u0(mesh.num_nodes(), Ensemble<S>(0.0));
  AssembledSystem<Ensemble<S>> a =
      enprop::assemble<Ensemble<S>>(ctx, field, PdeCoefficients{}, u0, std::span<const Ensemble<S>>(y));
  AssembledSystem<Ensemble<S>> b =
      enprop_b200::assemble<Ensemble<S>>(ctx, field, PdeCoefficients{}, u0, std::span<const Ensemble<S>>(y2));
  CHECK(same_bits(a.matrix.values, b.matrix.values) && same_bits(a.residual, b.residual));
  enprop::apply_dirichlet(a, mesh, DirichletBc{}, u0);
  DenseVector<Ensemble<S>> rhs(a.residual.size());
  for (size_t i = 0; i < rhs.size(); ++i) rhs[i] = -a.residual[i];
  SolverConfig cfg;
  cfg.tol = 1e-7;
  enprop::SolveResult<Ensemble<S>> r1 = enprop::pcg_solve(a.matrix, rhs, IdentityPreconditioner{}, cfg);
  enprop::SolveResult<Ensemble<S>> r2 = enprop_b200::pcg_solve(a.matrix, rhs, IdentityPreconditioner{}, cfg);
  CHECK(r1.iterations == r2.iterations && same_bits(r1.solution, r2.solution));
  bool inval = false;
  try {
    enprop_b200::pack_sample_group<Ensemble<S>>(pool2, 3 * S);
  } catch (const std::invalid_argument&) {
    inval = true;
  }
  CHECK(inval);
}

// newton_solve (fem.hpp:265-302) through the drop-in against the reference's
// own newton_solve (multigrid-preconditioned linear solves): iterate, steps,
// CG total and norms bit for bit
template <int S>
static void newton(int n, double beta) {
  StructuredMesh mesh(n);
  KlField field(3, 1.0, 0.1, 1.0);
  const PdeCoefficients coeffs{0.0, beta, {1.0, 0.0, 0.0}};
  const auto y = pack_sample_group<S>(draw_samples(7, S, 3), 0);
  NewtonOptions opt;
  opt.tol = 1e-8;
  opt.linear.tol = 1e-10;
  opt.multigrid.coarse_row_threshold = 100;
  enprop::NewtonResult<Ensemble<S>> ref = enprop::newton_solve<Ensemble<S>>(mesh, field, coeffs, y, DirichletBc{}, opt);
  enprop::NewtonResult<Ensemble<S>> r =
      enprop_b200::newton_solve(mesh, field, coeffs, y, DirichletBc{}, opt);
  CHECK(r.iterations == ref.iterations);
  CHECK(r.total_cg_iterations == ref.total_cg_iterations);
  CHECK(r.residual_norms == ref.residual_norms);
  CHECK(same_bits(r.solution, ref.solution));
}

int main() {
  spmv_dot_axpby<1>();
  spmv_dot_axpby<2>();
  spmv_dot_axpby<4>();
  spmv_dot_axpby<8>();
  spmv_dot_axpby<16>();
  spmv_dot_axpby<32>();
  for (int s : {1, 3, 4, 32}) spmv_outer_layout(s);

  for (int n : {1, 3, 9}) {
    std::vector<int> rm, ce;
    enprop_b200::build_node_graph(n, rm, ce);
    const Graph g = build_node_graph(StructuredMesh(n));
    CHECK(rm == g.row_map && ce == g.col_entry);
  }

  assembly_and_cg<double>(6);
  assembly_and_cg<Ensemble<4>>(6);
  assembly_and_cg<Ensemble<32>>(5);
  uncoupled_is_per_sample_scalar<8>(7);
  value_forms_and_samples<4>(5);
  value_forms_and_samples<32>(4);
  newton<4>(5, 0.0);
  newton<4>(5, 0.7);
  newton<1>(6, 0.7);

  // iteration exhaustion throws the reference's SolverError with the history
  // (test_pcg.cpp:164-179)
  std::mt19937_64 r3(3u);
  auto spd = testutil::random_spd_crs(r3, 50, 0.1);
  std::vector<double> b(50);
  for (auto& v : b) v = testutil::uniform_pm1(r3);
  SolverConfig cfg;
  cfg.tol = 1e-15;
  cfg.max_iterations = 2;
  bool thrown = false;
  try {
    enprop_b200::pcg_solve(spd, b, IdentityPreconditioner{}, cfg);
  } catch (const enprop::SolverError& err) {
    thrown = true;
    CHECK(err.history().size() == 3);
    CHECK(err.history().front() == 1.0);
  }
  CHECK(thrown);
  // shape errors are std::invalid_argument (kernels.hpp:17-18)
  bool inval = false;
  try {
    enprop_b200::spmv(crs_identity<double>(3), DenseVector<double>(2));
  } catch (const std::invalid_argument&) {
    inval = true;
  }
  CHECK(inval);

  std::printf("%s: %d checks, %d failures\n", g_fail ? "FAILED" : "ALL PASS", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
