// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the UNMODIFIED reference (/root/reference/proj/include/porofeti/*.hpp,
// compiled against the Eigen-API shim in eigen_shim/) on small cases and
// prints its outputs, so the oracle restatement (oracle/src) and the B200
// engine can be pinned to the reference itself.  Built by oracle/ref/Makefile
// into oracle/_ref/ref_driver (git-ignored); oracle/ref/make_ref_golden.py
// turns its output into tests/golden/ref_*.npz.
//
//   ref_driver <case> [steps_to_dump]
//
// Cases (all through the reference's own build_discretization
// (timeloop.hpp:51), StepSolver::advance (timeloop.hpp:150), FetiOperator
// (feti.hpp:74) and verify.hpp):
//   c1-schur / c1-generalized / c1-monolithic : BASELINE config 1 (mesh 32,
//       P1, E=1, nu=0.3, c0=1e-3, dt=1e-2, T=0.05, tol 1e-10) with the
//       time-linear manufactured solution of SURVEY App. C D7 supplied as a
//       reference Scenario (model.hpp:113-135);
//   mms-m<N> : the reference's own mms scenario (model.hpp:146), P2,
//       default_params (E=1e4, nu=0.2, c0=0.1), dt=1e-4, T=1e-2 (its defaults);
//   bm-m<N>  : the reference's Barry-Mercer scenario (model.hpp:274), P2,
//       default_params, dt=1e-2.
//
// Output: one line per array, "name n v0 v1 ..." (%.17g), scalars as n=1.
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <random>
#include <string>

#include "porofeti/timeloop.hpp"
#include "porofeti/verify.hpp"

using namespace porofeti;

namespace {

void put(const std::string& name, const Vector& v) {
  std::printf("%s %ld", name.c_str(), static_cast<long>(v.size()));
  for (Eigen::Index i = 0; i < v.size(); ++i) std::printf(" %.17g", v[i]);
  std::printf("\n");
}
void put(const std::string& name, double v) { std::printf("%s 1 %.17g\n", name.c_str(), v); }
void put(const std::string& name, const std::vector<double>& v) {
  std::printf("%s %zu", name.c_str(), v.size());
  for (double x : v) std::printf(" %.17g", x);
  std::printf("\n");
}

/// BASELINE configs 1-4 manufactured solution: u_P = t (S, S),
/// p = t S, S = sin(pi x) sin(pi y); u_E = u_P + (0, -gamma p (y - 1/2)),
/// gamma = alpha / (lambda_P + 2 mu_P); forcing from the strong form.
Scenario time_linear_mms(const ModelParams& P) {
  using std::numbers::pi;
  Scenario sc;
  sc.name = "mms-t";
  sc.rect_P = {0.0, 0.0, 1.0, 0.5};
  sc.rect_E = {0.0, 0.5, 1.0, 1.0};
  sc.interface_y = 0.5;
  const double muP = P.mu_P, laP = P.lambda_P, muE = P.mu_E, laE = P.lambda_E, al = P.alpha;
  const double G = laP + 2.0 * muP, gam = al / G;
  const double kk = P.K(0, 0), muf = P.mu_f, c0 = P.c0;
  auto S = [](const Vec2& x) { return std::sin(pi * x.x()) * std::sin(pi * x.y()); };
  ExactSolution ex;
  ex.u_P = [S](const Vec2& x, double t) { return Vec2(t * S(x), t * S(x)); };
  ex.u_E = [S, gam](const Vec2& x, double t) { return Vec2(t * S(x), t * S(x) - gam * t * S(x) * (x.y() - 0.5)); };
  ex.p = [S](const Vec2& x, double t) { return t * S(x); };
  sc.exact = ex;
  sc.f_P = [=](const Vec2& x, double t) {
    const double cp = std::cos(pi * (x.x() + x.y())), cm = std::cos(pi * (x.x() - x.y()));
    const double common = -pi * laP * cp + pi * muP * (cm - 2.0 * cp);
    return Vec2(pi * t * (al * std::sin(pi * x.y()) * std::cos(pi * x.x()) + common),
                pi * t * (al * std::sin(pi * x.x()) * std::cos(pi * x.y()) + common));
  };
  sc.f_E = [=](const Vec2& x, double t) {
    const double cx = std::cos(pi * x.x()), sx = std::sin(pi * x.x());
    const double cy = std::cos(pi * x.y()), sy = std::sin(pi * x.y());
    const double cp = std::cos(pi * (x.x() + x.y())), cm = std::cos(pi * (x.x() - x.y()));
    const double y2 = 2.0 * x.y() - 1.0;
    const double f0 = laE * (pi * al * y2 * cx * cy + 2.0 * al * sy * cx - 2.0 * pi * G * cp) +
                      muE * (pi * al * y2 * cx * cy + 2.0 * al * sy * cx + 2.0 * pi * G * (cm - 2.0 * cp));
    const double f1 = -laE * (pi * al * y2 * sx * sy - 4.0 * al * sx * cy + 2.0 * pi * G * cp) -
                      muE * (3.0 * pi * al * y2 * sx * sy - 8.0 * al * sx * cy + 2.0 * pi * G * (-cm + 2.0 * cp));
    return Vec2(pi * t * f0 / (2.0 * G), pi * t * f1 / (2.0 * G));
  };
  sc.z_source = [=](const Vec2& x, double t) {
    return c0 * S(x) + pi * al * std::sin(pi * (x.x() + x.y())) + 2.0 * pi * pi * (kk / muf) * t * S(x);
  };
  sc.u_bc_P = ex.u_P;
  sc.u_bc_E = ex.u_E;
  sc.p_bc = ex.p;
  auto zv = [](const Vec2&, double) { return Vec2::Zero().eval(); };
  auto zs = [](const Vec2&, double) { return 0.0; };
  sc.traction_P = zv, sc.traction_E = zv, sc.flux_zw = zs;
  sc.u0_P = zv, sc.u0_E = zv, sc.p0 = zs, sc.div_u0_P = zs, sc.div_u0_E = zs;
  sc.tag_rule_P = [](const Vec2& m) -> std::optional<FacetTag> {
    if (std::abs(m.y() - 0.5) < 1e-9) return FacetTag::interface();
    return FacetTag::dirichlet_displacement(FacetTag::Pressure::dirichlet);
  };
  sc.tag_rule_E = [](const Vec2& m) -> std::optional<FacetTag> {
    if (std::abs(m.y() - 0.5) < 1e-9) return FacetTag::interface();
    return FacetTag::dirichlet_displacement();
  };
  return sc;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver <c1-schur|c1-generalized|c1-monolithic|mms-m<N>|bm-m<N>> [dump_steps]\n");
    return 2;
  }
  const std::string cs = argv[1];
  int dump = argc > 2 ? std::atoi(argv[2]) : 1 << 30;
  ModelParams params;
  Scenario sc;
  int mesh_n = 32, order = 1;
  double T = 0.05, dt = 1e-2;
  SolveOptions opts;
  opts.tol = 1e-10;
  opts.max_iter = 500;
  opts.warm_start = true;
  if (cs.rfind("c1-", 0) == 0) {
    params = make_params(1.0, 0.3, 1.0, 0.3, 1.0, 1e-3, Mat2::Identity(), 1.0);
    sc = time_linear_mms(params);
    opts.solver = cs == "c1-schur"         ? SolverChoice::feti_schur
                  : cs == "c1-generalized" ? SolverChoice::feti_generalized
                                           : SolverChoice::monolithic;
  } else if (cs.rfind("mms-m", 0) == 0 || cs.rfind("bm-m", 0) == 0) {
    params = default_params();
    const bool mms = cs[0] == 'm';
    sc = mms ? mms_scenario(params) : barry_mercer_scenario(params);
    mesh_n = std::atoi(cs.c_str() + (mms ? 5 : 4));
    order = 2;
    T = mms ? sc.default_T : 3 * sc.default_dt;
    dt = sc.default_dt;
    opts.solver = SolverChoice::feti_schur;
  } else {
    std::fprintf(stderr, "unknown case %s\n", cs.c_str());
    return 2;
  }
  const TimeGrid grid = time_grid_from_dt(T, dt);
  const Discretization d = build_discretization(sc, params, mesh_n, order, grid);
  put("n_lambda", d.system.n_lambda);
  put("N", grid.N);
  put("dim_P", d.system.P.dim);
  put("dim_E", d.system.E.dim);
  const StepSolver solver(d, opts);
  if (const FetiOperator* op = solver.feti()) {
    // operator and preconditioner on lambda ~ U(-1,1), mt19937_64(20240901)
    std::mt19937_64 rng(20240901ull);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    Vector x(d.system.n_lambda);
    for (int i = 0; i < d.system.n_lambda; ++i) x[i] = U(rng);
    put("apply_in", x);
    put("apply_out", op->apply(x));
    put("precond_out", op->apply_preconditioner(x));
    // materialize_operator / materialize_preconditioner (feti.hpp:245-257),
    // column-major, for the small cases
    if (d.system.n_lambda <= 128) {
      const DenseMatrix Fm = materialize_operator(*op), Mm = materialize_preconditioner(*op);
      Vector f(Fm.rows() * Fm.cols()), m(Mm.rows() * Mm.cols());
      for (Eigen::Index k = 0; k < f.size(); ++k) f[k] = Fm.data()[k], m[k] = Mm.data()[k];
      put("F_dense", f);
      put("M_dense", m);
    }
    // the reference's operator on its own seeded check of the local factor (feti.hpp:28)
    Vector bp = Vector::Zero(d.system.P.dim);
    for (int i = 0; i < d.system.P.dim; ++i) bp[i] = U(rng);
    put("local_in_P", bp);
    put("local_out_P", op->factor_P().solve(bp));
  }
  StateSnapshot s = project_initial(d);
  double linf_u = 0.0, linf_p = 0.0;
  for (int n = 1; n <= grid.N; ++n) {
    PcgReport rep;
    s = solver.advance(s, &rep);
    const std::string k = std::to_string(n);
    if (n <= dump) {
      put("iters" + k, rep.iterations);
      put("rel" + k, rep.rel_residual);
      put("hist" + k, rep.residual_history);
      put("u_P" + k, s.u_P);
      put("eta" + k, s.eta);
      put("xi_P" + k, s.xi_P);
      put("p" + k, s.p);
      put("u_E" + k, s.u_E);
      put("xi_E" + k, s.xi_E);
      put("lambda" + k, s.lambda);
    }
    if (d.scenario.exact) {
      const double eu = snapshot_u_error(d, s), ep = snapshot_p_error(d, s);
      linf_u = std::max(linf_u, eu), linf_p = std::max(linf_p, ep);
      if (n <= dump) put("err_u" + k, eu), put("err_p" + k, ep);
    }
  }
  put("steps_run", grid.N);
  if (d.scenario.exact) put("linf_err_u", linf_u), put("linf_err_p", linf_p);
  return 0;
}
