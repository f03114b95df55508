// porofeti_b200.hpp — header-only C++ shim that re-creates the reference's
// FETI entry points (/root/reference/proj/include/porofeti/feti.hpp and
// timeloop.hpp) on top of the C ABI in porofeti_b200.h.  Eigen is not used:
// vectors are std::vector<double>.  Errors are rethrown as the reference's
// exception types (core.hpp:32-75).
//
//   reference                                   shim
//   porofeti::build_discretization + StepSolver  porofeti_b200::Problem(cfg)
//   FetiOperator::apply (feti.hpp:101)           Problem::apply
//   FetiOperator::apply_preconditioner (:127)    Problem::apply_preconditioner
//   FetiOperator::interface_rhs (:147)           Problem::interface_rhs
//   SubdomainFactorization::solve (:38)          Problem::local_solve
//   FetiOperator::back_substitute (:158)         Problem::back_substitute
//   FetiOperator::set_precond (:97)              Problem::set_precond
//   feti_pcg (:263)                              feti_pcg(Problem&, ...)
//   unpack_state (:443) / StateSnapshot fields   Problem::field
//   assemble_rhs_step loads (assembly.hpp:550)   Problem::set_loads
//   StepSolver::advance (timeloop.hpp:150)       StepSolver::advance
//   run_simulation (timeloop.hpp:206)            run_simulation
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#include <limits>
#include <cmath>
#include <algorithm>
#include <utility>

#include "porofeti_b200.h"

namespace porofeti_b200 {

using Vector = std::vector<double>;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularSubproblemError : Error {
  using Error::Error;
};
struct PcgBreakdownError : Error {
  using Error::Error;
};
struct SolverError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};

inline void check(int code, const pf_ctx* ctx) {
  if (code == PF_OK) return;
  const std::string msg = pf_last_error(ctx);
  switch (code) {
    case PF_SINGULAR: throw SingularSubproblemError(msg);
    case PF_BREAKDOWN: throw PcgBreakdownError(msg);
    case PF_NOT_CONVERGED: throw SolverError(msg);
    case PF_INVALID: throw ConfigError(msg);
    case PF_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

/// Reference PcgReport (feti.hpp:59-67).
struct PcgReport {
  int step = 0, iterations = 0;
  bool converged = false;
  double rel_residual = 0.0, seconds = 0.0;
  double true_residual = 0.0;  // ||P(rhs - F lambda)|| / ||r0||, recomputed at exit
};

inline PcgReport to_report(const pf_report& r) {
  return PcgReport{r.step, r.iterations, r.converged != 0, r.rel_residual, r.seconds, r.true_residual};
}

/// every ABI call reads / writes exactly n values: refuse a mismatched buffer
inline void check_size(const std::vector<double>& v, long long n, const char* what) {
  if ((long long)v.size() != n)
    throw ConfigError(std::string(what) + ": expected " + std::to_string(n) + " values, got " +
                      std::to_string(v.size()));
}

/// Reference StateSnapshot (state.hpp:8-12): per-subdomain saddle vectors
/// ([u, eta, xi, p] / [u, xi]) concatenated, plus the multiplier.
struct StateSnapshot {
  int step = 0;
  Vector x;
  Vector lambda;
};

inline pf_config default_config() {
  pf_config c{};
  c.mesh_n = 32, c.SX = 1, c.SY = 2, c.order = 1;
  c.E = 1.0, c.nu = 0.3, c.alpha = 1.0, c.c0 = 1e-3, c.kperm = 1.0, c.mu_f = 1.0, c.dt = 1e-2;
  c.steps = 5, c.mu_conv = 0, c.scenario = PF_SCEN_MMS_T, c.precond = PF_PREC_DIRICHLET;
  c.krylov = PF_KRYLOV_AUTO, c.tol = 1e-10, c.max_iter = 500, c.warm = 1, c.threads = 0;
  c.seed = 20240901ull, c.logk_mean = -2.0, c.logk_sd = 1.0;
  return c;
}

/// Reference SolverChoice (timeloop.hpp:113): feti-generalized and
/// feti-schur select the FETI preconditioner (the Krylov method follows the
/// multiplier layout); monolithic selects the direct interface solve, the
/// device analogue of MonolithicSolver (feti.hpp:313-440): the same discrete
/// solution without Krylov iterations (dense, n_lambda <= 65536).
enum class SolverChoice { feti_generalized, feti_schur, monolithic };

inline const char* solver_name(SolverChoice s) {
  switch (s) {
    case SolverChoice::feti_generalized: return "feti-generalized";
    case SolverChoice::feti_schur: return "feti-schur";
    default: return "monolithic";
  }
}

/// cfg.precond / cfg.krylov for a reference SolverChoice (the mortar-scaled
/// Dirichlet preconditioner on partitions with more than two subdomains)
inline void apply_solver_choice(pf_config& c, SolverChoice s) {
  const bool multi = c.SX * c.SY > 2;
  if (s == SolverChoice::monolithic) {
    c.krylov = PF_KRYLOV_DIRECT;
    if (c.precond == PF_PREC_IDENTITY) c.precond = multi ? PF_PREC_DIRICHLET_MORTAR : PF_PREC_DIRICHLET;
    return;
  }
  c.krylov = PF_KRYLOV_AUTO;
  if (s == SolverChoice::feti_schur) c.precond = multi ? PF_PREC_DIRICHLET_MORTAR : PF_PREC_DIRICHLET;
  else c.precond = multi ? PF_PREC_GENERALIZED_MORTAR : PF_PREC_GENERALIZED;
}

/// Reference SolveOptions (timeloop.hpp:123-131), same fields and defaults.
/// `parallel` has no meaning here (every subdomain runs in one launch);
/// `stride` and `verbose` belong to the caller's output loop.
struct SolveOptions {
  SolverChoice solver = SolverChoice::feti_generalized;
  double tol = 1e-8;
  int max_iter = 500;
  bool warm_start = true;
  bool parallel = true;
  int stride = 1;
  bool verbose = false;
};

/// cfg with the reference's SolveOptions applied (solver choice, tolerance,
/// iteration cap, warm start): what build_discretization + StepSolver(d, opts)
/// fix in the reference is fixed at Problem construction here.
inline pf_config with_options(pf_config c, const SolveOptions& o) {
  apply_solver_choice(c, o.solver);
  c.tol = o.tol, c.max_iter = o.max_iter, c.warm = o.warm_start ? 1 : 0;
  return c;
}

/// Discretisation + FETI operator living on the device.
class Problem {
 public:
  explicit Problem(const pf_config& cfg) { check(pf_create(&ctx_, &cfg), nullptr); refresh(); }
  /// build_discretization(scenario, ...) + StepSolver(d, opts) of the reference in one object
  Problem(const pf_config& cfg, const SolveOptions& opts) : Problem(with_options(cfg, opts)) {}
  ~Problem() { pf_destroy(ctx_); }
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;

  int n_lambda() const { return info_.n_lambda; }
  const pf_info& info() const { return info_; }
  pf_ctx* handle() const { return ctx_; }

  Vector apply(const Vector& x) const {
    check_size(x, info_.n_lambda, "apply");
    Vector y(info_.n_lambda);
    check(pf_apply(ctx_, x.data(), y.data()), ctx_);
    return y;
  }
  Vector apply_preconditioner(const Vector& r) const {
    check_size(r, info_.n_lambda, "apply_preconditioner");
    Vector z(info_.n_lambda);
    check(pf_apply_precond(ctx_, r.data(), z.data()), ctx_);
    return z;
  }
  Vector interface_rhs() const {
    Vector F(info_.n_lambda);
    check(pf_interface_rhs(ctx_, F.data()), ctx_);
    return F;
  }
  Vector local_solve(int s, Vector b) const {
    pf_sub_info si{};
    check(pf_get_sub_info(ctx_, s, &si), ctx_);
    check_size(b, si.dim, "local_solve");
    check(pf_local_solve(ctx_, s, b.data()), ctx_);
    return b;
  }
  /// StepSolver::advance on the device-resident state (one time step)
  PcgReport step() {
    pf_report r{};
    check(pf_step(ctx_, &r), ctx_);
    return to_report(r);
  }
  /// FetiOperator::set_precond (feti.hpp:97), PF_PREC_* kinds
  void set_precond(int kind) { check(pf_set_precond(ctx_, kind), ctx_); }
  /// FetiOperator::back_substitute (feti.hpp:158) for the current right-hand
  /// side: every subdomain's saddle vector, concatenated
  Vector back_substitute(const Vector& lambda) const {
    check_size(lambda, info_.n_lambda, "back_substitute");
    Vector x(info_.total_dim);
    check(pf_back_substitute(ctx_, lambda.data(), x.data()), ctx_);
    return x;
  }
  /// one named field (state.hpp:8-12) of subdomain s, or of all subdomains (s = -1)
  Vector field(int field, int s = -1) const {
    const int n = pf_field_size(ctx_, field, s);
    if (n < 0) throw ConfigError("field: not available for this subdomain");
    Vector out(n);
    check(pf_get_field(ctx_, field, s, out.data()), ctx_);
    return out;
  }
  /// caller-supplied loads for the next step (assembly.hpp:475-479 StepLoads + essential values)
  void set_loads(const Vector& F_u, const Vector& Z, const Vector& g, bool persistent = false) {
    long long nF = 0, nZ = 0, nG = 0;
    check(pf_load_sizes(ctx_, &nF, &nZ, &nG), ctx_);
    check_size(F_u, nF, "set_loads: F_u"), check_size(Z, nZ, "set_loads: Z"), check_size(g, nG, "set_loads: g");
    check(pf_set_loads(ctx_, F_u.data(), Z.data(), g.data(), persistent ? 1 : 0), ctx_);
  }
  /// snapshot_u_error / snapshot_p_error (verify.hpp:62-74) of the current state
  std::pair<double, double> errors() const {
    double eu = 0.0, ep = 0.0;
    check(pf_errors(ctx_, &eu, &ep), ctx_);
    return {eu, ep};
  }
  /// min / max nodal Darcy pressure of the current state (oscillation_check input)
  std::pair<double, double> pressure_range() const {
    double lo = 0.0, hi = 0.0;
    check(pf_pressure_range(ctx_, &lo, &hi), ctx_);
    return {lo, hi};
  }

 private:
  void refresh() { check(pf_get_info(ctx_, &info_), ctx_); }
  pf_ctx* ctx_ = nullptr;
  pf_info info_{};
};

/// Reference feti_pcg (feti.hpp:263-308): Krylov solve of the interface
/// problem for a caller right-hand side; throws SolverError when max_iter is
/// reached, PcgBreakdownError on breakdown.  residual_history as in REF.
struct PcgResult {
  Vector lambda;
  PcgReport report;
  std::vector<double> residual_history;
};
inline PcgResult feti_pcg(Problem& p, const Vector& rhs, const Vector& lambda_init, double tol, int max_iter) {
  check_size(rhs, p.n_lambda(), "feti_pcg: rhs");
  check_size(lambda_init, p.n_lambda(), "feti_pcg: lambda_init");
  PcgResult out;
  out.lambda.resize(p.n_lambda());
  pf_report r{};
  check(pf_krylov(p.handle(), rhs.data(), lambda_init.data(), tol, max_iter, out.lambda.data(), &r), p.handle());
  out.report = to_report(r);
  const int n = pf_last_history(p.handle(), nullptr, 0);
  out.residual_history.resize(n > 0 ? n : 0);
  if (n > 0) pf_last_history(p.handle(), out.residual_history.data(), n);
  return out;
}

/// Reference StepSolver (timeloop.hpp:135-193).
class StepSolver {
 public:
  explicit StepSolver(Problem& p) : p_(&p) {}
  /// reference signature StepSolver(d, opts): the options were applied when the
  /// Problem was built (Problem(cfg, opts)); kept for source compatibility
  StepSolver(Problem& p, const SolveOptions&) : p_(&p) {}
  StateSnapshot advance(const StateSnapshot& prev, PcgReport* report = nullptr) const {
    check_size(prev.x, p_->info().total_dim, "advance: prev.x");
    check_size(prev.lambda, p_->n_lambda(), "advance: prev.lambda");
    StateSnapshot next;
    next.x.resize(p_->info().total_dim);
    next.lambda.resize(p_->n_lambda());
    pf_report r{};
    check(pf_advance(p_->handle(), prev.x.data(), prev.lambda.data(), prev.step, next.x.data(), next.lambda.data(), &r),
          p_->handle());
    next.step = r.step;
    if (report) *report = to_report(r);
    return next;
  }

 private:
  Problem* p_;
};

/// Reference run_simulation (timeloop.hpp:206-221) on the device-resident state.
inline std::vector<PcgReport> run_simulation(Problem& p) {
  std::vector<PcgReport> out;
  for (int n = 0; n < p.info().N; ++n) {
    pf_report r{};
    check(pf_step(p.handle(), &r), p.handle());
    out.push_back(to_report(r));
  }
  return out;
}

/// Reference OscillationReport / oscillation_check (verify.hpp:160-195) on the
/// per-snapshot pressure ranges (Problem::pressure_range after each step).
struct OscillationReport {
  bool pass = true;
  double min_p = 0.0, max_p = 0.0, lower_bound = 0.0, upper_bound = 0.0, worst_violation = 0.0;
};
inline OscillationReport oscillation_check(const std::vector<std::pair<double, double>>& ranges,
                                           double max_boundary, double delta) {
  OscillationReport rep;
  rep.lower_bound = -delta, rep.upper_bound = max_boundary + delta;
  rep.min_p = std::numeric_limits<double>::infinity(), rep.max_p = -std::numeric_limits<double>::infinity();
  for (const auto& r : ranges) rep.min_p = std::min(rep.min_p, r.first), rep.max_p = std::max(rep.max_p, r.second);
  if (!std::isfinite(rep.min_p)) rep.min_p = rep.max_p = 0.0;
  double worst = 0.0;
  if (rep.min_p < rep.lower_bound && rep.lower_bound - rep.min_p > worst)
    worst = rep.lower_bound - rep.min_p, rep.worst_violation = rep.min_p, rep.pass = false;
  if (rep.max_p > rep.upper_bound && rep.max_p - rep.upper_bound > worst)
    rep.worst_violation = rep.max_p, rep.pass = false;
  return rep;
}

}  // namespace porofeti_b200
