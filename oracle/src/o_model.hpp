// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// o_model.hpp — restatement of model.hpp: Lame constants (:24-32), kappas
// (:38-42), ModelParams (:44-90) and scenarios.  Scenarios:
//   "mms"          reference stationary MMS (model.hpp:146-269), 2 subdomains
//   "barry-mercer" reference Barry-Mercer layout (model.hpp:274-324)
//   "mms-t"        BASELINE configs 1-4: time-linear MMS
//   "injection"    BASELINE config 5
#pragma once

#include <functional>

#include "o_mesh.hpp"

namespace oracle {

constexpr double kPi = 3.14159265358979323846;

enum class MuConv { paper, standard };

struct Params {
  double E_P = 1e4, nu_P = 0.2, E_E = 1e4, nu_E = 0.2;
  double lam_P = 0, mu_P = 0, lam_E = 0, mu_E = 0;
  double alpha = 1.0, c0 = 0.1;
  double K00 = 1, K01 = 0, K11 = 1;
  double mu_f = 1.0;
  double k1 = 0, k2 = 0, k3 = 0;
  MuConv conv = MuConv::paper;
};

inline void lame(double E, double nu, MuConv conv, double& lam, double& mu) {
  if (E <= 0) throw Error("lame_from_young_poisson: E must be positive");
  if (nu < 0 || nu >= 0.5) throw Error("lame_from_young_poisson: need 0 <= nu < 0.5");
  lam = E * nu / ((1 + nu) * (1 - 2 * nu));
  mu = conv == MuConv::paper ? E / (1 + nu) : E / (2 * (1 + nu));
}

inline Params make_params(double E_P, double nu_P, double E_E, double nu_E, double alpha, double c0,
                          double kperm, double mu_f, MuConv conv = MuConv::paper) {
  Params p;
  p.E_P = E_P, p.nu_P = nu_P, p.E_E = E_E, p.nu_E = nu_E;
  lame(E_P, nu_P, conv, p.lam_P, p.mu_P);
  lame(E_E, nu_E, conv, p.lam_E, p.mu_E);
  p.alpha = alpha;
  p.c0 = c0;
  if (!(kperm > 0)) throw Error("make_params: permeability tensor must be positive definite");
  p.K00 = p.K11 = kperm;
  p.K01 = 0;
  if (!(mu_f > 0)) throw Error("make_params: fluid viscosity must be positive");
  p.mu_f = mu_f;
  const double den = alpha * alpha + c0 * p.lam_P;
  if (den <= 0) throw Error("derived_kappas: alpha^2 + c0*lambda_P must be positive");
  p.k1 = alpha / den;
  p.k2 = p.lam_P / den;
  p.k3 = c0 / den;
  p.conv = conv;
  return p;
}

using SFn = std::function<double(const V2&, double)>;
using VFn = std::function<V2(const V2&, double)>;

struct Scenario {
  std::string name;
  VFn f_P, f_E;
  SFn z;                       // volumetric source (ignored where z_elem is set)
  VFn u_bc_P, u_bc_E;
  SFn p_bc;
  VFn tr_P, tr_E;
  SFn flux;
  VFn u0_P, u0_E;
  SFn p0, divu0_P, divu0_E;
  // exact fields for error sanity (optional)
  VFn ex_u_P, ex_u_E;
  SFn ex_p;
  // outer-boundary tag for an edge with midpoint m in region r
  std::function<Tag(Region, const V2&)> outer_tag;
  bool per_element = false;    // injection: z and K given per global element
  double src_x = 0.5, src_y = 0.25, src_r = 0.02, src_rate = 1.0;
};

inline bool near(double a, double b) { return std::abs(a - b) < 1e-9; }

inline VFn zero_v() {
  return [](const V2&, double) { return V2(0, 0); };
}
inline SFn zero_s() {
  return [](const V2&, double) { return 0.0; };
}

/// Stationary reference MMS: u = sin2pix sin2piy (both comps), p = sinpix sinpiy,
/// E-side correction -gamma p (y-1/2) on u_2 (model.hpp:146-269).
inline Scenario mms_stationary(const Params& P) {
  Scenario sc;
  sc.name = "mms";
  const double muP = P.mu_P, laP = P.lam_P, muE = P.mu_E, laE = P.lam_E, al = P.alpha;
  const double gam = al / (laP + 2 * muP);
  auto s = [](const V2& x) { return std::sin(2 * kPi * x.x) * std::sin(2 * kPi * x.y); };
  auto sx = [](const V2& x) { return 2 * kPi * std::cos(2 * kPi * x.x) * std::sin(2 * kPi * x.y); };
  auto sy = [](const V2& x) { return 2 * kPi * std::sin(2 * kPi * x.x) * std::cos(2 * kPi * x.y); };
  auto cc = [](const V2& x) { return std::cos(2 * kPi * x.x) * std::cos(2 * kPi * x.y); };
  auto pf = [](const V2& x) { return std::sin(kPi * x.x) * std::sin(kPi * x.y); };
  auto px = [](const V2& x) { return kPi * std::cos(kPi * x.x) * std::sin(kPi * x.y); };
  auto py = [](const V2& x) { return kPi * std::sin(kPi * x.x) * std::cos(kPi * x.y); };
  auto pxy = [](const V2& x) { return kPi * kPi * std::cos(kPi * x.x) * std::cos(kPi * x.y); };
  auto pxx = [pf](const V2& x) { return -kPi * kPi * pf(x); };
  auto ddiv = [s, cc](const V2& x) { return 4 * kPi * kPi * (cc(x) - s(x)); };
  auto deps = [s, cc](const V2& x) { return 2 * kPi * kPi * (cc(x) - 3 * s(x)); };
  auto corr = [pf, gam](const V2& x) { return -gam * pf(x) * (x.y - 0.5); };
  auto corr_y = [py, pf, gam](const V2& x) { return -gam * (py(x) * (x.y - 0.5) + pf(x)); };
  auto corr_xx = [pxx, gam](const V2& x) { return -gam * pxx(x) * (x.y - 0.5); };
  auto corr_xy = [pxy, px, gam](const V2& x) { return -gam * (pxy(x) * (x.y - 0.5) + px(x)); };
  auto corr_yy = [pxx, py, gam](const V2& x) { return -gam * (pxx(x) * (x.y - 0.5) + 2 * py(x)); };
  sc.ex_u_P = [s](const V2& x, double) { return V2(s(x), s(x)); };
  sc.ex_u_E = [s, corr](const V2& x, double) { return V2(s(x), s(x) + corr(x)); };
  sc.ex_p = [pf](const V2& x, double) { return pf(x); };
  sc.f_P = [=](const V2& x, double) {
    const double de = deps(x);
    return V2(-2 * muP * de + al * px(x) - laP * ddiv(x), -2 * muP * de + al * py(x) - laP * ddiv(x));
  };
  sc.f_E = [=](const V2& x, double) {
    const double de = deps(x);
    return V2(-2 * muE * (de + 0.5 * corr_xy(x)) - laE * (ddiv(x) + corr_xy(x)),
              -2 * muE * (de + 0.5 * corr_xx(x) + corr_yy(x)) - laE * (ddiv(x) + corr_yy(x)));
  };
  const double K00 = P.K00, K01 = P.K01, K11 = P.K11, muf = P.mu_f;
  sc.z = [=](const V2& x, double) {
    return -(K00 * pxx(x) + 2 * K01 * pxy(x) + K11 * pxx(x)) / muf;
  };
  sc.u_bc_P = sc.ex_u_P;
  sc.u_bc_E = sc.ex_u_E;
  sc.p_bc = sc.ex_p;
  sc.tr_P = sc.tr_E = zero_v();
  sc.flux = zero_s();
  sc.u0_P = sc.ex_u_P;
  sc.u0_E = sc.ex_u_E;
  sc.p0 = sc.ex_p;
  sc.divu0_P = [sx, sy](const V2& x, double) { return sx(x) + sy(x); };
  sc.divu0_E = [sx, sy, corr_y](const V2& x, double) { return sx(x) + sy(x) + corr_y(x); };
  sc.outer_tag = [](Region r, const V2&) {
    return r == Region::P ? Tag::clamp(PTag::dirichlet) : Tag::clamp();
  };
  return sc;
}

/// BASELINE configs 1-4: u_P = t(S,S), p = tS, S = sin pi x sin pi y;
/// u_E = u_P + (0, -gamma p (y-1/2)); forcing from the closed forms derived
/// with sympy.  Zero initial state, zero outer data.
inline Scenario mms_time_linear(const Params& P) {
  Scenario sc;
  sc.name = "mms-t";
  const double muP = P.mu_P, laP = P.lam_P, muE = P.mu_E, laE = P.lam_E, al = P.alpha;
  const double G = laP + 2 * muP, gam = al / G;
  const double kk = P.K00, muf = P.mu_f, c0 = P.c0;
  auto S = [](const V2& x) { return std::sin(kPi * x.x) * std::sin(kPi * x.y); };
  sc.ex_u_P = [S](const V2& x, double t) { return V2(t * S(x), t * S(x)); };
  sc.ex_u_E = [S, gam](const V2& x, double t) {
    return V2(t * S(x), t * S(x) - gam * t * S(x) * (x.y - 0.5));
  };
  sc.ex_p = [S](const V2& x, double t) { return t * S(x); };
  sc.f_P = [=](const V2& x, double t) {
    const double cp = std::cos(kPi * (x.x + x.y)), cm = std::cos(kPi * (x.x - x.y));
    const double common = -kPi * laP * cp + kPi * muP * (cm - 2 * cp);
    return V2(kPi * t * (al * std::sin(kPi * x.y) * std::cos(kPi * x.x) + common),
              kPi * t * (al * std::sin(kPi * x.x) * std::cos(kPi * x.y) + common));
  };
  sc.f_E = [=](const V2& x, double t) {
    const double cx = std::cos(kPi * x.x), sx = std::sin(kPi * x.x);
    const double cy = std::cos(kPi * x.y), sy = std::sin(kPi * x.y);
    const double cp = std::cos(kPi * (x.x + x.y)), cm = std::cos(kPi * (x.x - x.y));
    const double y2 = 2 * x.y - 1;
    const double f0 = laE * (kPi * al * y2 * cx * cy + 2 * al * sy * cx - 2 * kPi * G * cp) +
                      muE * (kPi * al * y2 * cx * cy + 2 * al * sy * cx + 2 * kPi * G * (cm - 2 * cp));
    const double f1 = -laE * (kPi * al * y2 * sx * sy - 4 * al * sx * cy + 2 * kPi * G * cp) -
                      muE * (3 * kPi * al * y2 * sx * sy - 8 * al * sx * cy + 2 * kPi * G * (-cm + 2 * cp));
    return V2(kPi * t * f0 / (2 * G), kPi * t * f1 / (2 * G));
  };
  sc.z = [=](const V2& x, double t) {
    return c0 * S(x) + kPi * al * std::sin(kPi * (x.x + x.y)) + 2 * kPi * kPi * (kk / muf) * t * S(x);
  };
  sc.u_bc_P = sc.ex_u_P;
  sc.u_bc_E = sc.ex_u_E;
  sc.p_bc = sc.ex_p;
  sc.tr_P = sc.tr_E = zero_v();
  sc.flux = zero_s();
  sc.u0_P = sc.u0_E = zero_v();
  sc.p0 = sc.divu0_P = sc.divu0_E = zero_s();
  sc.outer_tag = [](Region r, const V2&) {
    return r == Region::P ? Tag::clamp(PTag::dirichlet) : Tag::clamp();
  };
  return sc;
}

/// BASELINE config 5: zero forcing, zero Dirichlet u (all outer) and p (P outer),
/// constant-rate source on elements whose centroid is within src_r of (0.5,0.25).
inline Scenario injection(const Params&) {
  Scenario sc;
  sc.name = "injection";
  sc.f_P = sc.f_E = zero_v();
  sc.z = zero_s();
  sc.u_bc_P = sc.u_bc_E = zero_v();
  sc.p_bc = zero_s();
  sc.tr_P = sc.tr_E = zero_v();
  sc.flux = zero_s();
  sc.u0_P = sc.u0_E = zero_v();
  sc.p0 = sc.divu0_P = sc.divu0_E = zero_s();
  sc.outer_tag = [](Region r, const V2&) {
    return r == Region::P ? Tag::clamp(PTag::dirichlet) : Tag::clamp();
  };
  sc.per_element = true;
  return sc;
}

/// Reference Barry-Mercer layout (model.hpp:274-324): periodic pressure load
/// sin(t) on 0.2<=x<=0.8 of the drained bottom edge.
inline Scenario barry_mercer(const Params& P) {
  Scenario sc;
  sc.name = "barry-mercer";
  auto p2 = [](const V2& x, double t) { return (x.x >= 0.2 && x.x <= 0.8) ? std::sin(t) : 0.0; };
  sc.f_P = sc.f_E = zero_v();
  sc.z = zero_s();
  sc.u_bc_P = sc.u_bc_E = zero_v();
  sc.p_bc = [p2](const V2& x, double t) { return near(x.y, 0.0) ? p2(x, t) : 0.0; };
  const double al = P.alpha;
  sc.tr_P = [p2, al](const V2& x, double t) {
    return near(x.y, 0.0) ? V2(0, al * p2(x, t)) : V2(0, 0);
  };
  sc.tr_E = zero_v();
  sc.flux = zero_s();
  sc.u0_P = sc.u0_E = zero_v();
  sc.p0 = sc.divu0_P = sc.divu0_E = zero_s();
  sc.outer_tag = [](Region r, const V2& m) {
    if (r == Region::P) {
      if (near(m.y, 0.0)) return Tag{2u, PTag::dirichlet, false};
      return Tag{1u, PTag::dirichlet, false};
    }
    if (near(m.y, 1.0)) return Tag{2u, PTag::none, false};
    return Tag{1u, PTag::none, false};
  };
  return sc;
}

inline Scenario scenario_by_name(const std::string& n, const Params& P) {
  if (n == "mms") return mms_stationary(P);
  if (n == "mms-t") return mms_time_linear(P);
  if (n == "injection") return injection(P);
  if (n == "barry-mercer") return barry_mercer(P);
  throw ConfigError("unknown scenario '" + n + "'");
}

/// Portable per-element log-normal permeability:
/// splitmix64 stream -> Box-Muller (cos branch), log10 K ~ N(mean, sd),
/// global element order e = 2*(J*n + I) + k.
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return ((double)(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

inline std::vector<double> lognormal_permeability(int mesh_n, uint64_t seed, double mean, double sd) {
  SplitMix64 g(seed);
  std::vector<double> k(std::size_t(2) * mesh_n * mesh_n);
  for (auto& v : k) {
    const double u1 = g.uniform(), u2 = g.uniform();
    const double n = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    v = std::pow(10.0, mean + sd * n);
  }
  return k;
}

}  // namespace oracle
