// enprop_b200 C++ drop-in for the reference library's hot path (enprop,
// /root/reference/proj/include/enprop). Header-only, C++17; links against
// libenprop_b200.so through the C ABI in <enprop_b200.h>.
//
// The function templates take the reference's own types by structure — any
// matrix with num_rows / num_cols / row_map / col_entry / values, any vector
// that is a contiguous std::vector of `double` or of `Ensemble<S>` (a POD of
// S doubles, ensemble.hpp:30-106) — so a call site switches by replacing the
// namespace:
//
//     enprop::spmv(a, x, z);              ->  enprop_b200::spmv(a, x, z);
//     enprop::assemble(ctx, kl, c, u, y, sys)  -> enprop_b200::assemble(...);
//     enprop::pcg_solve(a, b, IdentityPreconditioner{}, cfg)
//                                          ->  enprop_b200::pcg_solve(a, b, IdentityPreconditioner{}, cfg);
//
// Semantics follow the reference exactly: same argument meaning, same output
// sizing, std::invalid_argument on shape errors, a SolverError carrying the
// residual history on non-convergence / indefinite operators. Results are
// bitwise equal to the reference for assembly, Dirichlet, SpMV, axpby, and —
// with the default DotOrder::serial — for dot/norm2 and pcg_solve as well.
// DotOrder::canonical selects the fast fixed-tree reduction.
//
// Host vectors are staged to the device per call (this is the compatibility
// path); the device-resident pipeline for throughput is enprop_problem_* in
// <enprop_b200.h>.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "enprop_b200.h"

// Result / system types: when the reference's headers are on the include path
// the drop-in returns the reference's own types (enprop::SolveResult<S>,
// enprop::AssembledSystem<S>, enprop::NewtonResult<S>), so call sites such as
//     enprop::SolveResult<E> r = enprop_b200::pcg_solve(...);
// compile unchanged; otherwise structurally identical local types are used.
#if !defined(ENPROP_B200_STANDALONE_TYPES) && __has_include("enprop/pcg.hpp") && __has_include("enprop/fem.hpp")
#include "enprop/fem.hpp"
#include "enprop/pcg.hpp"
#define ENPROP_B200_REFERENCE_TYPES 1
#endif

namespace enprop_b200 {

#ifdef ENPROP_B200_REFERENCE_TYPES
template <class Scalar>
using SolveResult = ::enprop::SolveResult<Scalar>;
template <class Scalar>
using AssembledSystem = ::enprop::AssembledSystem<Scalar>;
template <class Scalar>
using NewtonResult = ::enprop::NewtonResult<Scalar>;
#else
/// Same fields as enprop::SolveResult<Scalar> (pcg.hpp:33-38).
template <class Scalar>
struct SolveResult {
  std::vector<Scalar> solution;
  int iterations = 0;
  std::vector<double> residual_history;
};
/// Same fields as enprop::CrsMatrix<Scalar> (crs.hpp:19-69).
template <class Scalar>
struct CrsMatrix {
  int num_rows = 0, num_cols = 0;
  std::vector<int> row_map, col_entry;
  std::vector<Scalar> values;
};
/// Same fields as enprop::AssembledSystem<Scalar> (fem.hpp:34-38).
template <class Scalar>
struct AssembledSystem {
  CrsMatrix<Scalar> matrix;
  std::vector<Scalar> residual;
};
/// Same fields as enprop::NewtonResult<Scalar> (fem.hpp:251-257).
template <class Scalar>
struct NewtonResult {
  std::vector<Scalar> solution;
  int iterations = 0;
  int total_cg_iterations = 0;
  std::vector<double> residual_norms;
};
#endif

#ifndef ENPROP_B200_SOLVER_ERROR
/// Thrown like enprop::SolverError (pcg.hpp:22-31). Define
/// ENPROP_B200_SOLVER_ERROR to the reference's type (e.g. enprop::SolverError)
/// before including this header to throw that type instead.
class SolverError : public std::runtime_error {
 public:
  SolverError(const std::string& what, std::vector<double> history)
      : std::runtime_error(what), history_(std::move(history)) {}
  const std::vector<double>& history() const { return history_; }

 private:
  std::vector<double> history_;
};
#define ENPROP_B200_SOLVER_ERROR ::enprop_b200::SolverError
#endif

/// Error from the CUDA runtime / device (there is no CPU fallback).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

enum class DotOrder { serial = ENPROP_DOT_SERIAL, canonical = ENPROP_DOT_CANONICAL };

namespace detail {

inline void check(int rc, const char* what) {
  if (rc == ENPROP_OK) return;
  std::string msg = std::string(what) + ": " + enprop_last_error();
  if (rc == ENPROP_ERR_INVALID) throw std::invalid_argument(msg);
  throw DeviceError(msg);
}

struct Runtime {
  enprop_ctx* ctx = nullptr;
  DotOrder order = DotOrder::serial;
  Runtime() { check(enprop_ctx_create(0, &ctx), "enprop_ctx_create"); }
  ~Runtime() { enprop_ctx_destroy(ctx); }
  static Runtime& get() {
    thread_local Runtime rt;
    return rt;
  }
};

/// Device buffer owned for the duration of one call.
class Buf {
 public:
  Buf() = default;
  explicit Buf(size_t bytes) { check(enprop_malloc(Runtime::get().ctx, bytes, &p_), "enprop_malloc"); }
  Buf(const void* host, size_t bytes) : Buf(bytes) { up(host, bytes); }
  Buf(Buf&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
  Buf& operator=(Buf&& o) noexcept {
    std::swap(p_, o.p_);
    return *this;
  }
  ~Buf() {
    if (p_) enprop_free(Runtime::get().ctx, p_);
  }
  void up(const void* host, size_t bytes) {
    if (bytes) check(enprop_memcpy_h2d(Runtime::get().ctx, p_, host, bytes), "enprop_memcpy_h2d");
  }
  void down(void* host, size_t bytes) const {
    if (bytes) check(enprop_memcpy_d2h(Runtime::get().ctx, host, p_, bytes), "enprop_memcpy_d2h");
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
};

/// Ensemble width of a scalar type: double -> 1, Ensemble<S> (S doubles) -> S.
template <class Scalar>
constexpr int width() {
  static_assert(std::is_trivially_copyable_v<Scalar>, "scalar must be a POD of doubles");
  static_assert(sizeof(Scalar) % sizeof(double) == 0, "scalar must be a POD of doubles");
  return static_cast<int>(sizeof(Scalar) / sizeof(double));
}

template <class Vec>
using scalar_of = typename Vec::value_type;

template <class Scalar>
const double* raw(const std::vector<Scalar>& v) {
  return reinterpret_cast<const double*>(v.data());
}
template <class Scalar>
double* raw(std::vector<Scalar>& v) {
  return reinterpret_cast<double*>(v.data());
}

template <class Matrix>
struct DeviceCrs {
  Buf row_map, col_entry, values;
  explicit DeviceCrs(const Matrix& a)
      : row_map(a.row_map.data(), a.row_map.size() * sizeof(int)),
        col_entry(a.col_entry.data(), a.col_entry.size() * sizeof(int)),
        values(a.values.data(), a.values.size() * sizeof(scalar_of<decltype(a.values)>)) {}
};

}  // namespace detail

/// Reduction order used by dot / norm2 / pcg_solve of this thread.
inline void set_dot_order(DotOrder order) { detail::Runtime::get().order = order; }
inline DotOrder dot_order() { return detail::Runtime::get().order; }

// --------------------------------------------------------------------- SpMV
/// z = A x (kernels.hpp:15-26). z is resized to num_rows.
template <class Matrix, class Vector>
void spmv(const Matrix& a, const Vector& x, Vector& z) {
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  if (static_cast<int>(x.size()) != a.num_cols)
    throw std::invalid_argument("spmv: x length must equal num_cols");
  z.resize(a.num_rows);
  if (a.num_rows == 0) return;
  detail::DeviceCrs<Matrix> da(a);
  detail::Buf dx(x.data(), x.size() * sizeof(Scalar));
  detail::Buf dz(z.size() * sizeof(Scalar));
  detail::check(enprop_spmv(detail::Runtime::get().ctx, s, a.num_rows, a.num_cols,
                            da.row_map.template as<int>(), da.col_entry.template as<int>(),
                            da.values.template as<double>(), dx.as<double>(), dz.as<double>()),
                "spmv");
  dz.down(z.data(), z.size() * sizeof(Scalar));
}

template <class Matrix, class Vector>
Vector spmv(const Matrix& a, const Vector& x) {
  Vector z;
  spmv(a, x, z);
  return z;
}

/// z = A x on the sample-major layout (spmv_outer, kernels.hpp:38-56): any
/// matrix with num_rows / num_cols / ensemble_size / row_map / col_entry /
/// values (OuterEnsembleMatrix, crs.hpp:138-147). z is resized to
/// num_rows * ensemble_size.
template <class OuterMatrix>
void spmv_outer(const OuterMatrix& a, const std::vector<double>& x, std::vector<double>& z) {
  const long long nnz = static_cast<long long>(a.col_entry.size());
  const long long cols = static_cast<long long>(a.num_cols);
  if (static_cast<long long>(x.size()) != cols * a.ensemble_size)
    throw std::invalid_argument("spmv_outer: x length must equal num_cols*ensemble_size");
  z.resize(static_cast<std::size_t>(a.num_rows) * a.ensemble_size);
  if (a.num_rows == 0 || a.ensemble_size == 0) return;
  detail::Buf rm(a.row_map.data(), a.row_map.size() * sizeof(int));
  detail::Buf ce(a.col_entry.data(), a.col_entry.size() * sizeof(int));
  detail::Buf va(a.values.data(), a.values.size() * sizeof(double));
  detail::Buf dx(x.data(), x.size() * sizeof(double));
  detail::Buf dz(z.size() * sizeof(double));
  detail::check(enprop_spmv_outer(detail::Runtime::get().ctx, a.ensemble_size, a.num_rows,
                                  a.num_cols, nnz, rm.as<int>(), ce.as<int>(), va.as<double>(),
                                  dx.as<double>(), dz.as<double>()),
                "spmv_outer");
  dz.down(z.data(), z.size() * sizeof(double));
}

// ------------------------------------------------------------- dot, axpby
/// Coupled inner product (kernels.hpp:62-69).
template <class Vector>
double dot(const Vector& u, const Vector& v) {
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  if (u.size() != v.size()) throw std::invalid_argument("dot: length mismatch");
  detail::Buf du(u.data(), u.size() * sizeof(Scalar)), dv(v.data(), v.size() * sizeof(Scalar));
  double out = 0.0;
  detail::check(enprop_dot(detail::Runtime::get().ctx, s, static_cast<int64_t>(u.size()),
                           du.as<double>(), &u == &v ? du.as<double>() : dv.as<double>(),
                           static_cast<int>(dot_order()), 0, nullptr, &out),
                "dot");
  return out;
}

template <class Vector>
double norm2(const Vector& u) {
  return std::sqrt(dot(u, u));
}

/// y = alpha*x + beta*y (kernels.hpp:78-85); Coef = double or Ensemble<S>.
template <class Coef, class Vector>
void axpby(const Coef& alpha, const Vector& x, const Coef& beta, Vector& y) {
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  constexpr int cw = detail::width<Coef>();
  static_assert(cw == 1 || cw == s, "axpby: coefficients must be scalars or per-lane ensembles");
  if (x.size() != y.size()) throw std::invalid_argument("axpby: length mismatch");
  detail::Buf dx(x.data(), x.size() * sizeof(Scalar)), dy(y.data(), y.size() * sizeof(Scalar));
  detail::check(enprop_axpby(detail::Runtime::get().ctx, s, static_cast<int64_t>(x.size()), cw != 1,
                             reinterpret_cast<const double*>(&alpha), dx.as<double>(),
                             reinterpret_cast<const double*>(&beta), dy.as<double>()),
                "axpby");
  dy.down(y.data(), y.size() * sizeof(Scalar));
}

// ------------------------------------------------------------------ samples
/// draw_samples (samples.cpp:7-18): count vectors of m coordinates uniform in
/// [-1, 1), bitwise the reference's mt19937_64 sequence.
inline std::vector<std::vector<double>> draw_samples(std::uint64_t seed, int count, int m) {
  std::vector<double> flat(static_cast<size_t>(count > 0 ? count : 0) * (m > 0 ? m : 0));
  detail::check(enprop_draw_samples(seed, count, m, flat.data()), "draw_samples");
  std::vector<std::vector<double>> out(count);
  for (int i = 0; i < count; ++i) out[i].assign(flat.begin() + (size_t)i * m, flat.begin() + (size_t)(i + 1) * m);
  return out;
}

/// pack_sample_group<Ensemble> (samples.hpp:18-31): out[j][e] = samples[group_start + e][j];
/// Scalar is the reference's Ensemble<S> (or any POD of S doubles).
template <class Scalar>
std::vector<Scalar> pack_sample_group(const std::vector<std::vector<double>>& samples, int group_start = 0) {
  constexpr int s = detail::width<Scalar>();
  if (group_start < 0 || group_start + s > static_cast<int>(samples.size()))
    throw std::invalid_argument("pack_sample_group: not enough samples for the group");
  const size_t m = samples[group_start].size();
  std::vector<double> flat(samples.size() * m);
  for (size_t i = 0; i < samples.size(); ++i) {
    if (samples[i].size() != m && static_cast<int>(i) >= group_start && static_cast<int>(i) < group_start + s)
      throw std::invalid_argument("pack_sample_group: sample lengths differ");
    for (size_t j = 0; j < m && j < samples[i].size(); ++j) flat[i * m + j] = samples[i][j];
  }
  std::vector<Scalar> out(m);
  detail::check(enprop_pack_sample_group(flat.data(), static_cast<int>(samples.size()), static_cast<int>(m),
                                         group_start, s, reinterpret_cast<double*>(out.data())),
                "pack_sample_group");
  return out;
}

// -------------------------------------------------------- mesh and assembly
/// build_node_graph(StructuredMesh(n)) (mesh.cpp:13-55), bit-exact.
inline void build_node_graph(int cells_per_axis, std::vector<int>& row_map,
                             std::vector<int>& col_entry) {
  if (cells_per_axis < 1) throw std::invalid_argument("StructuredMesh: cells_per_axis must be at least 1");
  const int64_t rows = static_cast<int64_t>(cells_per_axis + 1) * (cells_per_axis + 1) * (cells_per_axis + 1);
  const int64_t nnz = enprop_mesh_nnz(cells_per_axis);
  detail::Buf rm((rows + 1) * sizeof(int)), ce(nnz * sizeof(int));
  detail::check(enprop_build_node_graph(detail::Runtime::get().ctx, cells_per_axis, rm.as<int>(),
                                        ce.as<int>()),
                "build_node_graph");
  row_map.resize(rows + 1);
  col_entry.resize(nnz);
  rm.down(row_map.data(), row_map.size() * sizeof(int));
  ce.down(col_entry.data(), col_entry.size() * sizeof(int));
}

namespace detail {
template <class Field>
enprop_kl_params kl_of(const Field& f) {
  return enprop_kl_params{f.num_terms(), f.mean(), f.sigma(), f.correlation_length()};
}
template <class Coeffs>
enprop_pde_coeffs coeffs_of(const Coeffs& c) {
  enprop_pde_coeffs o{c.alpha, c.beta, {c.velocity[0], c.velocity[1], c.velocity[2]}};
  return o;
}
}  // namespace detail

/// assemble<Scalar> (fem.hpp:115-202). Ctx is enprop::AssemblyContext (or any
/// type with mesh().cells_per_axis()), Field an enprop::KlField, Coeffs an
/// enprop::PdeCoefficients, System an enprop::AssembledSystem<Scalar>.
template <class Scalar, class Ctx, class Field, class Coeffs, class Samples, class System>
void assemble(const Ctx& actx, const Field& field, const Coeffs& coeffs, const std::vector<Scalar>& u,
              const Samples& samples, System& out) {
  constexpr int s = detail::width<Scalar>();
  const int n = actx.mesh().cells_per_axis();
  const int64_t rows = static_cast<int64_t>(n + 1) * (n + 1) * (n + 1);
  if (static_cast<int64_t>(u.size()) != rows)
    throw std::invalid_argument("assemble: solution vector length mismatch");
  if (static_cast<int>(samples.size()) != field.num_terms())
    throw std::invalid_argument("assemble: sample vector length mismatch");
  auto& ctx = detail::Runtime::get();
  const int64_t nnz = enprop_mesh_nnz(n);
  detail::Buf rm((rows + 1) * sizeof(int)), ce(nnz * sizeof(int));
  detail::check(enprop_build_node_graph(ctx.ctx, n, rm.as<int>(), ce.as<int>()), "assemble: graph");
  detail::Buf du(u.data(), u.size() * sizeof(Scalar));
  detail::Buf dy(samples.data(), samples.size() * sizeof(Scalar));
  detail::Buf dv(nnz * sizeof(Scalar)), dr(rows * sizeof(Scalar));
  const enprop_kl_params kl = detail::kl_of(field);
  const enprop_pde_coeffs co = detail::coeffs_of(coeffs);
  detail::check(enprop_assemble(ctx.ctx, s, n, &kl, &co, du.as<double>(), dy.as<double>(),
                                rm.as<int>(), dv.as<double>(), dr.as<double>(), nullptr),
                "assemble");
  out.matrix.num_rows = static_cast<int>(rows);
  out.matrix.num_cols = static_cast<int>(rows);
  out.matrix.row_map.resize(rows + 1);
  out.matrix.col_entry.resize(nnz);
  out.matrix.values.resize(nnz);
  out.residual.resize(rows);
  rm.down(out.matrix.row_map.data(), (rows + 1) * sizeof(int));
  ce.down(out.matrix.col_entry.data(), nnz * sizeof(int));
  dv.down(out.matrix.values.data(), nnz * sizeof(Scalar));
  dr.down(out.residual.data(), rows * sizeof(Scalar));
}

/// assemble<Scalar> returning the system by value (fem.hpp:204-210).
template <class Scalar, class Ctx, class Field, class Coeffs, class Samples>
AssembledSystem<Scalar> assemble(const Ctx& actx, const Field& field, const Coeffs& coeffs,
                                 const std::vector<Scalar>& u, const Samples& samples) {
  AssembledSystem<Scalar> out;
  assemble<Scalar>(actx, field, coeffs, u, samples, out);
  return out;
}

/// apply_dirichlet (fem.hpp:218-243) on a system assembled on `mesh`.
template <class System, class Mesh, class Bc, class Vector>
void apply_dirichlet(System& system, const Mesh& mesh, const Bc& bc, const Vector& u) {
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  const int n = mesh.cells_per_axis();
  if (static_cast<int>(u.size()) != mesh.num_nodes())
    throw std::invalid_argument("apply_dirichlet: solution vector length mismatch");
  auto& a = system.matrix;
  detail::Buf rm(a.row_map.data(), a.row_map.size() * sizeof(int));
  detail::Buf ce(a.col_entry.data(), a.col_entry.size() * sizeof(int));
  detail::Buf dv(a.values.data(), a.values.size() * sizeof(Scalar));
  detail::Buf dr(system.residual.data(), system.residual.size() * sizeof(Scalar));
  detail::Buf du(u.data(), u.size() * sizeof(Scalar));
  const enprop_dirichlet_bc b{bc.x0_value, bc.x1_value};
  detail::check(enprop_apply_dirichlet(detail::Runtime::get().ctx, s, n, &b, rm.as<int>(),
                                       ce.as<int>(), du.as<double>(), dv.as<double>(),
                                       dr.as<double>()),
                "apply_dirichlet");
  dv.down(a.values.data(), a.values.size() * sizeof(Scalar));
  dr.down(system.residual.data(), system.residual.size() * sizeof(Scalar));
}

// ------------------------------------------------------------------------ CG
/// pcg_solve (pcg.hpp:52-103) with the identity preconditioner (pcg.hpp:40-45):
/// coupled ensemble CG = pcg_solve<Ensemble<S>>; at S = 1, pcg_solve<double>.
/// Config is an enprop::SolverConfig (tol, max_iterations).
template <class Matrix, class Vector, class Precond, class Config>
SolveResult<detail::scalar_of<Vector>> pcg_solve(const Matrix& a, const Vector& b, Precond&&,
                                                 const Config& config) {
  static_assert(std::is_empty_v<std::decay_t<Precond>>,
                "enprop_b200 accelerates identity-preconditioned CG (IdentityPreconditioner); "
                "the multigrid preconditioner is out of scope");
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  if (a.num_rows != a.num_cols) throw std::invalid_argument("pcg_solve: matrix must be square");
  if (static_cast<int>(b.size()) != a.num_rows)
    throw std::invalid_argument("pcg_solve: right-hand side length mismatch");
  SolveResult<Scalar> result;
  result.solution.resize(b.size());
  detail::DeviceCrs<Matrix> da(a);
  detail::Buf db(b.data(), b.size() * sizeof(Scalar)), dx(b.size() * sizeof(Scalar));
  enprop_cg_options opt{ENPROP_CG_COUPLED, static_cast<int>(dot_order()), 0, config.tol,
                        config.max_iterations, 16};
  std::vector<double> hist(static_cast<size_t>(config.max_iterations) + 1);
  int iters = 0, status = 0, hlen = 0;
  const int rc = enprop_cg(detail::Runtime::get().ctx, s, a.num_rows, da.row_map.template as<int>(),
                           da.col_entry.template as<int>(), da.values.template as<double>(),
                           db.as<double>(), dx.as<double>(), &opt, &iters, &status, hist.data(), &hlen);
  hist.resize(hlen);
  if (rc == ENPROP_ERR_NO_CONVERGENCE || rc == ENPROP_ERR_INDEFINITE)
    throw ENPROP_B200_SOLVER_ERROR(enprop_last_error(), std::move(hist));
  detail::check(rc, "pcg_solve");
  dx.down(result.solution.data(), b.size() * sizeof(Scalar));
  result.iterations = iters;
  result.residual_history = std::move(hist);
  return result;
}

/// Per-sample ("uncoupled") ensemble CG: s independent pcg_solve<double> runs
/// on the extracted components (bench.cpp:340-349), fused in one pass over the
/// shared graph. Failing samples report a non-zero status instead of throwing.
template <class Scalar>
struct UncoupledResult {
  std::vector<Scalar> solution;
  std::vector<int> iterations;            // per sample
  std::vector<int> status;                // ENPROP_OK / NO_CONVERGENCE / INDEFINITE
  std::vector<std::vector<double>> residual_history;  // per sample
};

template <class Matrix, class Vector, class Config>
UncoupledResult<detail::scalar_of<Vector>> pcg_solve_uncoupled(const Matrix& a, const Vector& b,
                                                               const Config& config) {
  using Scalar = detail::scalar_of<Vector>;
  constexpr int s = detail::width<Scalar>();
  if (a.num_rows != a.num_cols) throw std::invalid_argument("pcg_solve: matrix must be square");
  if (static_cast<int>(b.size()) != a.num_rows)
    throw std::invalid_argument("pcg_solve: right-hand side length mismatch");
  UncoupledResult<Scalar> r;
  r.solution.resize(b.size());
  r.iterations.resize(s);
  r.status.resize(s);
  detail::DeviceCrs<Matrix> da(a);
  detail::Buf db(b.data(), b.size() * sizeof(Scalar)), dx(b.size() * sizeof(Scalar));
  enprop_cg_options opt{ENPROP_CG_UNCOUPLED, static_cast<int>(dot_order()), 0, config.tol,
                        config.max_iterations, 16};
  std::vector<double> hist((static_cast<size_t>(config.max_iterations) + 1) * s);
  std::vector<int> hlen(s);
  const int rc = enprop_cg(detail::Runtime::get().ctx, s, a.num_rows, da.row_map.template as<int>(),
                           da.col_entry.template as<int>(), da.values.template as<double>(),
                           db.as<double>(), dx.as<double>(), &opt, r.iterations.data(),
                           r.status.data(), hist.data(), hlen.data());
  if (rc != ENPROP_ERR_NO_CONVERGENCE && rc != ENPROP_ERR_INDEFINITE) detail::check(rc, "pcg_solve");
  dx.down(r.solution.data(), b.size() * sizeof(Scalar));
  r.residual_history.resize(s);
  for (int e = 0; e < s; ++e)
    for (int it = 0; it < hlen[e]; ++it) r.residual_history[e].push_back(hist[static_cast<size_t>(it) * s + e]);
  return r;
}

// ------------------------------------------------------------------ Newton
/// newton_solve (fem.hpp:265-302) on the device-resident problem
/// (enprop_problem_newton_mg): from u = 0, assemble residual + Jacobian at u,
/// impose Dirichlet, stop when the coupled residual norm falls below
/// options.tol times the first, else build the multigrid hierarchy of the
/// Jacobian (options.multigrid) and solve J du = -f by MG-preconditioned
/// coupled CG (options.linear), u = 1.0*du + 1.0*u -- the reference's own
/// algorithm, bitwise. Mesh is an enprop::StructuredMesh, Options an
/// enprop::NewtonOptions. Throws SolverError with the residual norms after
/// max_iterations steps.
template <class Scalar, class Mesh, class Field, class Coeffs, class Bc, class Options>
NewtonResult<Scalar> newton_solve(const Mesh& mesh, const Field& field, const Coeffs& coeffs,
                                  const std::vector<Scalar>& samples, const Bc& bc,
                                  const Options& options) {
  constexpr int s = detail::width<Scalar>();
  if (static_cast<int>(samples.size()) != field.num_terms())
    throw std::invalid_argument("newton_solve: sample vector length mismatch");
  auto& rt = detail::Runtime::get();
  enprop_problem_desc d{};
  d.cells_per_axis = mesh.cells_per_axis();
  d.ensemble_size = s;
  d.kl = detail::kl_of(field);
  d.coeffs = detail::coeffs_of(coeffs);
  d.bc = enprop_dirichlet_bc{bc.x0_value, bc.x1_value};
  enprop_problem* p = nullptr;
  detail::check(enprop_problem_create(rt.ctx, &d, &p), "newton_solve");
  std::unique_ptr<enprop_problem, int (*)(enprop_problem*)> guard(p, enprop_problem_destroy);
  detail::Buf dy(samples.data(), samples.size() * sizeof(Scalar));
  enprop_newton_options o{};
  o.tol = options.tol;
  o.max_iterations = options.max_iterations;
  o.linear = enprop_cg_options{ENPROP_CG_COUPLED, static_cast<int>(dot_order()), 0, options.linear.tol,
                               options.linear.max_iterations, 16};
  int steps = 0, cg_total = 0, nn = 0;
  std::vector<double> norms(static_cast<size_t>(options.max_iterations > 0 ? options.max_iterations : 0) + 1);
  const enprop_mg_options mo{options.multigrid.coarse_row_threshold, options.multigrid.chebyshev_degree,
                             options.multigrid.eigenvalue_ratio, options.multigrid.eigenvalue_boost,
                             options.multigrid.power_iterations};
  const int rc = enprop_problem_newton_mg(p, dy.as<double>(), &o, &mo, &steps, &cg_total, norms.data(), &nn);
  norms.resize(nn);
  if (rc == ENPROP_ERR_NO_CONVERGENCE || rc == ENPROP_ERR_INDEFINITE)
    throw ENPROP_B200_SOLVER_ERROR(enprop_last_error(), std::move(norms));
  detail::check(rc, "newton_solve");
  NewtonResult<Scalar> r;
  int rows = 0;
  double* x = nullptr;
  detail::check(enprop_problem_views(p, &rows, nullptr, nullptr, nullptr, nullptr, nullptr, &x), "newton_solve");
  r.solution.resize(rows);
  detail::check(enprop_memcpy_d2h(rt.ctx, r.solution.data(), x, static_cast<size_t>(rows) * sizeof(Scalar)),
                "newton_solve");
  r.iterations = steps;
  r.total_cg_iterations = cg_total;
  r.residual_norms = std::move(norms);
  return r;
}

}  // namespace enprop_b200
