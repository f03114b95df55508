// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// o_verify.hpp — restatement of verify.hpp:19-82: spatial L2 errors of a
// state against the scenario's exact solution (elementwise degree-4 Dunavant
// quadrature of (field_h - exact)^2, square root taken), the displacement
// error over the union of all subdomains and the Darcy-pressure error over
// the poroelastic ones, and the L-inf(L2) maximum over time levels.
#pragma once

#include <cmath>

#include "o_feti.hpp"

namespace oracle {

constexpr int kErrorQuadDegree = 4;  // verify.hpp:15

/// sum over the subdomain's triangles of int |u_h - u|^2 (l2_error_vector, verify.hpp:44-60)
inline double l2_error_vector_sq(const Sub& S, const Vec& x, const VFn& exact, double t, int order) {
  const Quad rule = triangle_rule(kErrorQuadDegree);
  double v[6];
  V2 g[6];
  double acc = 0.0;
  for (int tri = 0; tri < S.mesh.nt(); ++tri) {
    const auto c = S.mesh.coords(tri);
    const V2 e1 = c[1] - c[0], e2 = c[2] - c[0];
    const double det = e1.x * e2.y - e2.x * e1.y;
    const std::vector<int> nodes = detail::local_u_nodes(S.mesh, tri, order);
    for (int q = 0; q < rule.size(); ++q) {
      eval_basis(order, rule.pts[q], v, g);
      const V2 xq = c[0] + e1 * rule.pts[q].x + e2 * rule.pts[q].y;
      double hx = 0.0, hy = 0.0;
      for (std::size_t i = 0; i < nodes.size(); ++i) {
        hx += x[S.off_u + S.u.dof(nodes[i], 0)] * v[i];
        hy += x[S.off_u + S.u.dof(nodes[i], 1)] * v[i];
      }
      const V2 ex = exact(xq, t);
      acc += rule.w[q] * std::abs(det) * ((hx - ex.x) * (hx - ex.x) + (hy - ex.y) * (hy - ex.y));
    }
  }
  return acc;
}

/// sum over the subdomain's triangles of int (p_h - p)^2 (l2_error_scalar, verify.hpp:19-41)
inline double l2_error_scalar_sq(const Sub& S, const Vec& x, const SFn& exact, double t) {
  const Quad rule = triangle_rule(kErrorQuadDegree);
  double v[6];
  V2 g[6];
  double acc = 0.0;
  for (int tri = 0; tri < S.mesh.nt(); ++tri) {
    const auto c = S.mesh.coords(tri);
    const V2 e1 = c[1] - c[0], e2 = c[2] - c[0];
    const double det = e1.x * e2.y - e2.x * e1.y;
    for (int q = 0; q < rule.size(); ++q) {
      eval_basis(1, rule.pts[q], v, g);
      const V2 xq = c[0] + e1 * rule.pts[q].x + e2 * rule.pts[q].y;
      double h = 0.0;
      for (int i = 0; i < 3; ++i) h += x[S.off_p + S.mesh.tri[tri][i]] * v[i];
      const double d = h - exact(xq, t);
      acc += rule.w[q] * std::abs(det) * d * d;
    }
  }
  return acc;
}

/// snapshot_u_error / snapshot_p_error (verify.hpp:62-74) over all subdomains
inline void snapshot_errors(const Disc& D, const State& st, double& eu, double& ep) {
  if (!D.sc.ex_u_P || !D.sc.ex_u_E || !D.sc.ex_p)
    throw ConfigError("snapshot_errors: scenario '" + D.sc.name + "' has no exact solution");
  double su = 0.0, sp = 0.0;
  for (std::size_t s = 0; s < D.subs.size(); ++s) {
    const Sub& S = D.subs[s];
    const bool P = S.region == Region::P;
    su += l2_error_vector_sq(S, st.x[s], P ? D.sc.ex_u_P : D.sc.ex_u_E, st.t, S.u.order);
    if (P) sp += l2_error_scalar_sq(S, st.x[s], D.sc.ex_p, st.t);
  }
  eu = std::sqrt(su), ep = std::sqrt(sp);
}

}  // namespace oracle
