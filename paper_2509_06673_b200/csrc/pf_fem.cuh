// pf_fem.cuh — per-element sm_100a kernels: saddle assembly (K1) and the
// per-step right-hand side (K2).
//
// Element forms follow the reference elements.hpp:152-230 (degree-4 Dunavant
// rule, P1/P2 Lagrange bases, 2mu eps:eps, -psi div phi, mass, (1/mu_f) K
// grad.grad); assembly into the constrained saddle of assembly.hpp:338-398
// with the symmetric elimination of :246-271 (constrained rows skipped,
// free-row/constrained-column entries into the lifting matrix).  Elements are
// processed in 8 colours (cell parity x triangle) so no two concurrent
// threads touch the same node: deterministic without atomics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pf {
namespace dev {

// Dunavant degree-4 rule (published constants; reference elements.hpp:37-38)
__constant__ double c_qx[6] = {0.091576213509771, 0.816847572980459, 0.091576213509771,
                               0.445948490915965, 0.108103018168070, 0.445948490915965};
__constant__ double c_qy[6] = {0.091576213509771, 0.091576213509771, 0.816847572980459,
                               0.445948490915965, 0.445948490915965, 0.108103018168070};
__constant__ double c_qw[6] = {0.5 * 0.109951743655322, 0.5 * 0.109951743655322, 0.5 * 0.109951743655322,
                               0.5 * 0.223381589678011, 0.5 * 0.223381589678011, 0.5 * 0.223381589678011};

struct FemType {
  int region, n_u, n_s, dim, off_eta, off_xi, off_p;
  long long kptr, kcol, lptr, lcol, cpos, cons;  // offsets into concatenated type arrays
  int ncons;
};

struct FemSub {
  int type, sx, sy;
  double x0, y0, x1, y1;
  long long kval, lval, vec, zacc, gval;  // offsets: K values, lift values, saddle vectors, Z, g
};

struct FemSet {
  int cx, cy, order, nv, nsub, mesh_n, scenario;
  const int* tri;    // 3 per triangle (shared topology)
  const int* tedge;  // 3 per triangle
  const FemType* types;
  const FemSub* subs;
  const int *kptr, *kcol, *lptr, *lcol, *cpos;
  const int* cons;   // per type: (sidx, node, comp) triplets
  const double* kelem;
  const uint8_t* srcel;
  const double* cxy;  // constraint node coordinates (2 per constraint, at FemSub.gval)
  double lam_P, mu_P, lam_E, mu_E, alpha, c0, kperm, mu_f, k1, k2, k3, tau;
};

__device__ __forceinline__ void basis(int order, double x, double y, double* v, double* gx, double* gy) {
  const double l0 = 1.0 - x - y, l1 = x, l2 = y;
  if (order == 1) {
    v[0] = l0, v[1] = l1, v[2] = l2;
    gx[0] = -1, gy[0] = -1, gx[1] = 1, gy[1] = 0, gx[2] = 0, gy[2] = 1;
  } else {
    v[0] = l0 * (2 * l0 - 1);
    v[1] = l1 * (2 * l1 - 1);
    v[2] = l2 * (2 * l2 - 1);
    v[3] = 4 * l0 * l1;
    v[4] = 4 * l1 * l2;
    v[5] = 4 * l2 * l0;
    gx[0] = (4 * l0 - 1) * -1.0, gy[0] = (4 * l0 - 1) * -1.0;
    gx[1] = (4 * l1 - 1) * 1.0, gy[1] = (4 * l1 - 1) * 0.0;
    gx[2] = (4 * l2 - 1) * 0.0, gy[2] = (4 * l2 - 1) * 1.0;
    gx[3] = 4.0 * (l1 * -1.0 + l0 * 1.0), gy[3] = 4.0 * (l1 * -1.0 + l0 * 0.0);
    gx[4] = 4.0 * (l2 * 1.0 + l1 * 0.0), gy[4] = 4.0 * (l2 * 0.0 + l1 * 1.0);
    gx[5] = 4.0 * (l0 * 0.0 + l2 * -1.0), gy[5] = 4.0 * (l0 * 1.0 + l2 * -1.0);
  }
}

struct Elem {
  double ax, ay;                  // vertex 0
  double J00, J01, J10, J11, det;
  double I00, I01, I10, I11;      // J^{-T}
  int t, gl;                      // local triangle, global element id
  int v[3];
  int un[6];
};

__device__ __forceinline__ bool element_of(const FemSet& S, int color, int tid, int& sub, Elem& E) {
  const int pi = color & 1, pj = (color >> 1) & 1, tk = color >> 2;
  const int nci = (S.cx - pi + 1) / 2, ncj = (S.cy - pj + 1) / 2, per = nci * ncj;
  if (per == 0) return false;
  sub = tid / per;
  if (sub >= S.nsub) return false;
  const int r = tid % per;
  const int i = pi + 2 * (r % nci), j = pj + 2 * (r / nci);
  const FemSub& F = S.subs[sub];
  const double hx = (F.x1 - F.x0) / S.cx, hy = (F.y1 - F.y0) / S.cy;
  // reference vertex coordinates rect.x0 + i*hx (mesh.hpp:113-116)
  const double xa = F.x0 + i * hx, ya = F.y0 + j * hy;
  const double xb = F.x0 + (i + 1) * hx, yb = F.y0 + j * hy;
  const double xc = F.x0 + (i + 1) * hx, yc = F.y0 + (j + 1) * hy;
  const double xd = F.x0 + i * hx, yd = F.y0 + (j + 1) * hy;
  double p1x, p1y, p2x, p2y;
  if (tk == 0) p1x = xb, p1y = yb, p2x = xc, p2y = yc;
  else p1x = xc, p1y = yc, p2x = xd, p2y = yd;
  E.ax = xa, E.ay = ya;
  E.J00 = p1x - xa, E.J10 = p1y - ya, E.J01 = p2x - xa, E.J11 = p2y - ya;
  E.det = E.J00 * E.J11 - E.J01 * E.J10;
  E.I00 = E.J11 / E.det, E.I01 = -E.J10 / E.det, E.I10 = -E.J01 / E.det, E.I11 = E.J00 / E.det;
  E.t = 2 * (j * S.cx + i) + tk;
  E.gl = 2 * ((F.sy * S.cy + j) * S.mesh_n + (F.sx * S.cx + i)) + tk;
  for (int q = 0; q < 3; ++q) E.v[q] = S.tri[3 * E.t + q];
  E.un[0] = E.v[0], E.un[1] = E.v[1], E.un[2] = E.v[2];
  E.un[3] = S.nv + S.tedge[3 * E.t + 2];
  E.un[4] = S.nv + S.tedge[3 * E.t + 0];
  E.un[5] = S.nv + S.tedge[3 * E.t + 1];
  return true;
}

__device__ __forceinline__ int find_col(const int* col, int b, int e, int c) {
  while (b < e) {
    const int m = (b + e) >> 1;
    if (col[m] < c) b = m + 1;
    else e = m;
  }
  return b;
}

__device__ __forceinline__ void add_entry(const FemSet& S, const FemType& T, const FemSub& F, double* Kv, double* Lv,
                                          int r, int c, double v) {
  const int* cpos = S.cpos + T.cpos;
  if (cpos[r] >= 0) return;
  const int cc = cpos[c];
  if (cc < 0) {
    const int* kp = S.kptr + T.kptr;
    const int q = find_col(S.kcol + T.kcol, kp[r], kp[r + 1], c);
    Kv[F.kval + q] += v;
  } else {
    const int* lp = S.lptr + T.lptr;
    const int q = find_col(S.lcol + T.lcol, lp[r], lp[r + 1], cc);
    Lv[F.lval + q] += v;
  }
}

/// Geometry of an arbitrary triangle (AffineMap, elements.hpp:132-144): J =
/// [v1 - v0, v2 - v0], I = J^{-T}.
__device__ __forceinline__ void affine_map(const double* tri, Elem& E) {
  E.ax = tri[0], E.ay = tri[1];
  E.J00 = tri[2] - tri[0], E.J10 = tri[3] - tri[1], E.J01 = tri[4] - tri[0], E.J11 = tri[5] - tri[1];
  E.det = E.J00 * E.J11 - E.J01 * E.J10;
  E.I00 = E.J11 / E.det, E.I01 = -E.J10 / E.det, E.I10 = -E.J01 / E.det, E.I11 = E.J00 / E.det;
}

/// local_elastic_matrix (elements.hpp:152-175) entry block (i, j): the 2x2
/// component block 2 mu int eps(phi_i e_a) : eps(phi_j e_b), Dunavant degree 4
__device__ __forceinline__ void elastic_block(int order, const Elem& E, double mu, int i, int j, double& a00,
                                              double& a01, double& a10, double& a11) {
  double v[6], rgx[6], rgy[6];
  const double adet = fabs(E.det);
  a00 = a01 = a10 = a11 = 0.0;
  for (int q = 0; q < 6; ++q) {
    basis(order, c_qx[q], c_qy[q], v, rgx, rgy);
    const double gix = E.I00 * rgx[i] + E.I01 * rgy[i], giy = E.I10 * rgx[i] + E.I11 * rgy[i];
    const double gjx = E.I00 * rgx[j] + E.I01 * rgy[j], gjy = E.I10 * rgx[j] + E.I11 * rgy[j];
    const double w = 2.0 * mu * (c_qw[q] * adet);
    a00 += w * (gix * gjx + 0.5 * giy * gjy);
    a01 += w * 0.5 * giy * gjx;
    a10 += w * 0.5 * gix * gjy;
    a11 += w * (giy * gjy + 0.5 * gix * gjx);
  }
}

/// local_div_matrix (elements.hpp:178-197) entries (i, 2j), (i, 2j+1):
/// -int psi_i d_c phi_j
__device__ __forceinline__ void div_pair(int order, const Elem& E, int i, int j, double& bx, double& by) {
  double v[6], rgx[6], rgy[6], sv[3], sgx[3], sgy[3];
  const double adet = fabs(E.det);
  bx = by = 0.0;
  for (int q = 0; q < 6; ++q) {
    basis(order, c_qx[q], c_qy[q], v, rgx, rgy);
    basis(1, c_qx[q], c_qy[q], sv, sgx, sgy);
    const double gjx = E.I00 * rgx[j] + E.I01 * rgy[j], gjy = E.I10 * rgx[j] + E.I11 * rgy[j];
    const double w = c_qw[q] * adet;
    bx -= w * sv[i] * gjx;
    by -= w * sv[i] * gjy;
  }
}

/// local_mass_matrix (elements.hpp:199-212) and local_diffusion_matrix
/// (elements.hpp:215-230, isotropic K = kk I) entries (i, j)
__device__ __forceinline__ void mass_diffusion(const Elem& E, double kk, double mu_f, int i, int j, double& m,
                                               double& d) {
  double sv[3], sgx[3], sgy[3];
  const double adet = fabs(E.det);
  m = d = 0.0;
  for (int q = 0; q < 6; ++q) {
    basis(1, c_qx[q], c_qy[q], sv, sgx, sgy);
    const double w = c_qw[q] * adet;
    m += w * sv[i] * sv[j];
    const double gix = E.I00 * sgx[i] + E.I01 * sgy[i], giy = E.I10 * sgx[i] + E.I11 * sgy[i];
    const double gjx = E.I00 * sgx[j] + E.I01 * sgy[j], gjy = E.I10 * sgx[j] + E.I11 * sgy[j];
    d += (c_qw[q] * adet / mu_f) * ((kk * gjx) * gix + (kk * gjy) * giy);
  }
}

/// The element-level entry point (pf_local_matrices): the four local forms of
/// one triangle, thread per entry, by the same device functions the assembly
/// kernel uses.  Outputs row-major: elastic 2nb x 2nb, div 3 x 2nb, mass and
/// diffusion 3 x 3.
__global__ void k_local_forms(const double* tri, int order, double mu, double kk, double mu_f, double* elastic,
                              double* div, double* mass, double* diffusion) {
  Elem E;
  affine_map(tri, E);
  const int nb = order == 2 ? 6 : 3;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nb * nb) {
    const int i = t / nb, j = t % nb;
    double a00, a01, a10, a11;
    elastic_block(order, E, mu, i, j, a00, a01, a10, a11);
    const int n2 = 2 * nb;
    elastic[(2 * i) * n2 + 2 * j] = a00, elastic[(2 * i) * n2 + 2 * j + 1] = a01;
    elastic[(2 * i + 1) * n2 + 2 * j] = a10, elastic[(2 * i + 1) * n2 + 2 * j + 1] = a11;
  }
  if (t < 3 * nb) {
    const int i = t / nb, j = t % nb;
    double bx, by;
    div_pair(order, E, i, j, bx, by);
    div[i * 2 * nb + 2 * j] = bx, div[i * 2 * nb + 2 * j + 1] = by;
  }
  if (t < 9) {
    double m, d;
    mass_diffusion(E, kk, mu_f, t / 3, t % 3, m, d);
    mass[t] = m, diffusion[t] = d;
  }
}

/// K1: element assembly of one colour into the constrained saddles + lifting.
__global__ void k_assemble(FemSet S, int color, double* Kv, double* Lv) {
  int sub;
  Elem E;
  if (!element_of(S, color, blockIdx.x * blockDim.x + threadIdx.x, sub, E)) return;
  const FemSub& F = S.subs[sub];
  const FemType& T = S.types[F.type];
  const int nb = S.order == 2 ? 6 : 3;
  const bool P = T.region == 0;
  const double mu = P ? S.mu_P : S.mu_E;
  double kk = S.kperm;
  if (S.kelem) kk = S.kelem[E.gl];
  // elastic block and div block (elements.hpp:152-197)
  for (int i = 0; i < nb; ++i) {
    for (int j = 0; j < nb; ++j) {
      double a00, a01, a10, a11;
      elastic_block(S.order, E, mu, i, j, a00, a01, a10, a11);
      add_entry(S, T, F, Kv, Lv, 2 * E.un[i], 2 * E.un[j], a00);
      add_entry(S, T, F, Kv, Lv, 2 * E.un[i], 2 * E.un[j] + 1, a01);
      add_entry(S, T, F, Kv, Lv, 2 * E.un[i] + 1, 2 * E.un[j], a10);
      add_entry(S, T, F, Kv, Lv, 2 * E.un[i] + 1, 2 * E.un[j] + 1, a11);
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < nb; ++j) {
      double bx, by;
      div_pair(S.order, E, i, j, bx, by);
      const int si = T.off_xi + E.v[i];
      add_entry(S, T, F, Kv, Lv, si, 2 * E.un[j], bx);       // B
      add_entry(S, T, F, Kv, Lv, si, 2 * E.un[j] + 1, by);
      add_entry(S, T, F, Kv, Lv, 2 * E.un[j], si, bx);       // B^T
      add_entry(S, T, F, Kv, Lv, 2 * E.un[j] + 1, si, by);
    }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double m, d;
      mass_diffusion(E, kk, S.mu_f, i, j, m, d);
      const int vi = E.v[i], vj = E.v[j];
      if (P) {
        add_entry(S, T, F, Kv, Lv, T.off_eta + vi, T.off_eta + vj, S.k2 * m);
        add_entry(S, T, F, Kv, Lv, T.off_eta + vi, T.off_xi + vj, S.k1 * m);
        add_entry(S, T, F, Kv, Lv, T.off_eta + vi, T.off_p + vj, -m);
        add_entry(S, T, F, Kv, Lv, T.off_xi + vi, T.off_eta + vj, S.k1 * m);
        add_entry(S, T, F, Kv, Lv, T.off_xi + vi, T.off_xi + vj, -S.k3 * m);
        add_entry(S, T, F, Kv, Lv, T.off_p + vi, T.off_eta + vj, -m);
        add_entry(S, T, F, Kv, Lv, T.off_p + vi, T.off_p + vj, -S.tau * d);
      } else {
        add_entry(S, T, F, Kv, Lv, T.off_xi + vi, T.off_xi + vj, -(1.0 / S.lam_E) * m);
      }
    }
}

/// unit diagonal at constrained rows (assembly.hpp:266)
__global__ void k_constraint_diag(FemSet S, double* Kv) {
  const int sub = blockIdx.y;
  if (sub >= S.nsub) return;
  const FemSub& F = S.subs[sub];
  const FemType& T = S.types[F.type];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < T.ncons; k += gridDim.x * blockDim.x) {
    const int r = S.cons[T.cons + 3 * k];
    const int* kp = S.kptr + T.kptr;
    const int q = find_col(S.kcol + T.kcol, kp[r], kp[r + 1], r);
    Kv[F.kval + q] = 1.0;
  }
}

// ---------------------------------------------------------------------------
// Scenario closed forms (model.hpp:146-324 and SURVEY App. C D7/D8)
// ---------------------------------------------------------------------------
constexpr double kPiD = 3.14159265358979323846;

__device__ void body_force(const FemSet& S, bool P, double x, double y, double t, double& fx, double& fy) {
  fx = fy = 0.0;
  if (S.scenario == 0) {  // time-linear MMS
    const double muP = S.mu_P, laP = S.lam_P, muE = S.mu_E, laE = S.lam_E, al = S.alpha;
    if (P) {
      const double cp = cos(kPiD * (x + y)), cm = cos(kPiD * (x - y));
      const double common = -kPiD * laP * cp + kPiD * muP * (cm - 2 * cp);
      fx = kPiD * t * (al * sin(kPiD * y) * cos(kPiD * x) + common);
      fy = kPiD * t * (al * sin(kPiD * x) * cos(kPiD * y) + common);
    } else {
      const double G = laP + 2 * muP;
      const double cx = cos(kPiD * x), sx = sin(kPiD * x), cy = cos(kPiD * y), sy = sin(kPiD * y);
      const double cp = cos(kPiD * (x + y)), cm = cos(kPiD * (x - y));
      const double y2 = 2 * y - 1;
      const double f0 = laE * (kPiD * al * y2 * cx * cy + 2 * al * sy * cx - 2 * kPiD * G * cp) +
                        muE * (kPiD * al * y2 * cx * cy + 2 * al * sy * cx + 2 * kPiD * G * (cm - 2 * cp));
      const double f1 = -laE * (kPiD * al * y2 * sx * sy - 4 * al * sx * cy + 2 * kPiD * G * cp) -
                        muE * (3 * kPiD * al * y2 * sx * sy - 8 * al * sx * cy + 2 * kPiD * G * (-cm + 2 * cp));
      fx = kPiD * t * f0 / (2 * G);
      fy = kPiD * t * f1 / (2 * G);
    }
  } else if (S.scenario == 1) {  // reference stationary MMS
    const double muP = S.mu_P, laP = S.lam_P, muE = S.mu_E, laE = S.lam_E, al = S.alpha;
    const double gam = al / (laP + 2 * muP);
    const double s = sin(2 * kPiD * x) * sin(2 * kPiD * y), cc = cos(2 * kPiD * x) * cos(2 * kPiD * y);
    const double pf = sin(kPiD * x) * sin(kPiD * y);
    const double px = kPiD * cos(kPiD * x) * sin(kPiD * y), py = kPiD * sin(kPiD * x) * cos(kPiD * y);
    const double pxy = kPiD * kPiD * cos(kPiD * x) * cos(kPiD * y), pxx = -kPiD * kPiD * pf;
    const double ddiv = 4 * kPiD * kPiD * (cc - s), de = 2 * kPiD * kPiD * (cc - 3 * s);
    if (P) {
      fx = -2 * muP * de + al * px - laP * ddiv;
      fy = -2 * muP * de + al * py - laP * ddiv;
    } else {
      const double cxx = -gam * pxx * (y - 0.5), cxy = -gam * (pxy * (y - 0.5) + px);
      const double cyy = -gam * (pxx * (y - 0.5) + 2 * py);
      fx = -2 * muE * (de + 0.5 * cxy) - laE * (ddiv + cxy);
      fy = -2 * muE * (de + 0.5 * cxx + cyy) - laE * (ddiv + cyy);
    }
  }
}

__device__ double source_z(const FemSet& S, double x, double y, double t, int gl) {
  if (S.scenario == 0) {
    const double Sx = sin(kPiD * x) * sin(kPiD * y);
    return S.c0 * Sx + kPiD * S.alpha * sin(kPiD * (x + y)) + 2 * kPiD * kPiD * (S.kperm / S.mu_f) * t * Sx;
  }
  if (S.scenario == 1) {
    const double pxx = -kPiD * kPiD * sin(kPiD * x) * sin(kPiD * y);
    return -(S.kperm * pxx + S.kperm * pxx) / S.mu_f;
  }
  if (S.scenario == 2) return S.srcel[gl] ? 1.0 : 0.0;
  return 0.0;
}

/// displacement / pressure essential values at node (x, y)
__device__ void bc_values(const FemSet& S, bool P, double x, double y, double t, double& ux, double& uy, double& p) {
  ux = uy = p = 0.0;
  if (S.scenario == 0) {
    const double Sx = sin(kPiD * x) * sin(kPiD * y);
    ux = t * Sx, uy = t * Sx, p = t * Sx;
    if (!P) uy = t * Sx - (S.alpha / (S.lam_P + 2 * S.mu_P)) * t * Sx * (y - 0.5);
  } else if (S.scenario == 1) {
    const double s = sin(2 * kPiD * x) * sin(2 * kPiD * y), pf = sin(kPiD * x) * sin(kPiD * y);
    ux = s, uy = s, p = pf;
    if (!P) uy = s + -(S.alpha / (S.lam_P + 2 * S.mu_P)) * pf * (y - 0.5);
  } else if (S.scenario == 3) {
    p = (fabs(y) < 1e-9 && x >= 0.2 && x <= 0.8) ? sin(t) : 0.0;
  }
}

/// K2: element loads of one colour: b_u += int f phi, zacc += int z psi.
__global__ void k_rhs_elem(FemSet S, int color, double t, double* b, double* zacc) {
  int sub;
  Elem E;
  if (!element_of(S, color, blockIdx.x * blockDim.x + threadIdx.x, sub, E)) return;
  const FemSub& F = S.subs[sub];
  const FemType& T = S.types[F.type];
  const bool P = T.region == 0;
  const int nb = S.order == 2 ? 6 : 3;
  const double adet = fabs(E.det);
  double v[6], gx[6], gy[6], sv[3], sgx[3], sgy[3];
  double Fx[6] = {0, 0, 0, 0, 0, 0}, Fy[6] = {0, 0, 0, 0, 0, 0}, Z[3] = {0, 0, 0};
  for (int q = 0; q < 6; ++q) {
    basis(S.order, c_qx[q], c_qy[q], v, gx, gy);
    const double x = E.ax + E.J00 * c_qx[q] + E.J01 * c_qy[q];
    const double y = E.ay + E.J10 * c_qx[q] + E.J11 * c_qy[q];
    double fx, fy;
    body_force(S, P, x, y, t, fx, fy);
    const double w = c_qw[q] * adet;
    for (int i = 0; i < nb; ++i) Fx[i] += w * v[i] * fx, Fy[i] += w * v[i] * fy;
    if (P) {
      basis(1, c_qx[q], c_qy[q], sv, sgx, sgy);
      const double zq = source_z(S, x, y, t, E.gl);
      for (int i = 0; i < 3; ++i) Z[i] += w * sv[i] * zq;
    }
  }
  double* bb = b + F.vec;
  for (int i = 0; i < nb; ++i) bb[2 * E.un[i]] += Fx[i], bb[2 * E.un[i] + 1] += Fy[i];
  if (P)
    for (int i = 0; i < 3; ++i) zacc[F.zacc + E.v[i]] += Z[i];
}

/// constraint values g at time t (assembly.hpp:562-571)
__global__ void k_constraint_values(FemSet S, double t, double* g) {
  const int sub = blockIdx.y;
  if (sub >= S.nsub) return;
  const FemSub& F = S.subs[sub];
  const FemType& T = S.types[F.type];
  const double hx = (F.x1 - F.x0) / S.cx, hy = (F.y1 - F.y0) / S.cy;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < T.ncons; k += gridDim.x * blockDim.x) {
    const int node = S.cons[T.cons + 3 * k + 1], comp = S.cons[T.cons + 3 * k + 2];
    (void)node, (void)hx, (void)hy;
    const double x = S.cxy[2 * (F.gval + k)], y = S.cxy[2 * (F.gval + k) + 1];
    double ux, uy, p;
    bc_values(S, T.region == 0, x, y, t, ux, uy, p);
    g[F.gval + k] = comp == 0 ? ux : comp == 1 ? uy : p;
  }
}

}  // namespace dev
}  // namespace pf
