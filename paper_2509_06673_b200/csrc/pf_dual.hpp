// pf_dual.hpp — explicit local dual operators, host side.
//
// For every subdomain s with Dirichlet boundary set B (free interface trace
// dofs, SubType::Bset) and local multipliers (the rows of G_s):
//   F_s  = G_s K_s^+ G_s^T          (the subdomain's share of the F-apply),
//   Sd_s = G_s S_s G_s^T            (its share of the Dirichlet preconditioner),
// with S_s = K_BB - K_BI K_II^{-1} K_IB the Schur complement of the saddle
// onto B.  Both come out of ONE partial factorisation per subdomain of the
// bordered matrix
//        [ K_s   G_s^T ]      ordered [ interior (nested dissection) | B | multipliers ],
//        [ G_s   0     ]
// on the device multifrontal kernels (pf_factor.cuh): the root front (B and
// the multipliers, one dense supernode) holds [[S, G_B^T], [G_B, 0]] after the
// interior is eliminated; Sd_s = G_B S G_B^T is read from it, then eliminating
// the B pivots leaves -G_B S^{-1} G_B^T = -F_s in the multiplier block.
// Floating subdomains: K_s^+ is the fixing-dof generalised inverse of the
// sweep path (identity rows/columns, and the fixing dofs neither receive nor
// return values); the fixing dofs lie on interface sides (in B), so for F the
// root front gets S's fixing rows/columns -> identity and G's fixing columns
// -> 0 between the two reads (Sd keeps the unregularised S and full G).
#pragma once

#include <algorithm>
#include <map>

#include "pf_disc.hpp"
#include "pf_symbolic.hpp"

namespace pf {

struct DualType {
  bool ok = false;
  std::string why;             // reason when !ok (engine falls back to the sweeps)
  int dim = 0, nB = 0, nM = 0;  // root front order = nB + nM
  std::vector<int> bset;       // natural dof ids of B (root order)
  std::vector<int> fixpos;     // positions in B of the fixing dofs (floating)
  std::vector<int> g_j, g_b;   // G pattern: (local multiplier, B position), sorted by (j, b)
  std::vector<int> g_ptr;      // per local multiplier j: [g_ptr[j], g_ptr[j+1]) into g_j/g_b
  Csr A;                       // bordered pattern (dim + nM), natural order
  std::vector<int> kmap;       // per A entry: K value index (>= 0) or -2 - (G pattern index)
  SymFactor F;
  FrontMaps M;
  AScatter S;
  int root = -1;
};

/// local multipliers of a subdomain (sorted global ids) and its G entries as
/// (local multiplier, natural column, value)
inline void dual_local_mults(const Subdomain& S, std::vector<int>& lam, std::vector<std::tuple<int, int, double>>& ent) {
  lam.assign(S.g_lam.begin(), S.g_lam.end());
  std::sort(lam.begin(), lam.end());
  lam.erase(std::unique(lam.begin(), lam.end()), lam.end());
  ent.clear();
  for (std::size_t q = 0; q < S.g_lam.size(); ++q) {
    const int j = int(std::lower_bound(lam.begin(), lam.end(), S.g_lam[q]) - lam.begin());
    ent.emplace_back(j, S.g_col[q], S.g_val[q]);
  }
}

/// Build the bordered system of a type from one representative subdomain.
inline DualType build_dual_type(const SubType& T, const Subdomain& rep) {
  DualType X;
  X.dim = T.dim;
  X.bset = T.Bset;
  X.nB = (int)X.bset.size();
  std::vector<int> bpos(T.dim, -1);
  for (int i = 0; i < X.nB; ++i) bpos[X.bset[i]] = i;
  if (T.floating)
    for (int f : T.fix) {
      if (f < 0) continue;
      if (bpos[f] < 0) {
        X.why = "fixing dof outside the Dirichlet boundary set";
        return X;
      }
      X.fixpos.push_back(bpos[f]);
    }
  std::vector<int> lam;
  std::vector<std::tuple<int, int, double>> ent;
  dual_local_mults(rep, lam, ent);
  X.nM = (int)lam.size();
  if (!dev::dual_panel_width(X.nB + X.nM)) {  // k_dual_root stages a panel of the root front
    X.why = "root front exceeds the shared-memory panel of k_dual_root";
    return X;
  }
  std::vector<std::pair<int, int>> gp;
  for (auto& e : ent) {
    const int col = std::get<1>(e);
    if (bpos[col] < 0) {
      X.why = "multiplier column outside the Dirichlet boundary set";
      return X;
    }
    gp.emplace_back(std::get<0>(e), bpos[col]);
  }
  std::sort(gp.begin(), gp.end());
  if (std::adjacent_find(gp.begin(), gp.end()) != gp.end()) {
    X.why = "duplicate G entries";
    return X;
  }
  X.g_ptr.assign(X.nM + 1, 0);
  for (auto& e : gp) X.g_j.push_back(e.first), X.g_b.push_back(e.second), X.g_ptr[e.first + 1]++;
  for (int j = 0; j < X.nM; ++j) X.g_ptr[j + 1] += X.g_ptr[j];
  // bordered pattern
  const int n = T.dim + X.nM;
  std::vector<std::pair<int, int>> rc;
  rc.reserve(T.K.nnz() + 2 * gp.size() + X.nM);
  for (int i = 0; i < T.dim; ++i)
    for (int q = T.K.ptr[i]; q < T.K.ptr[i + 1]; ++q) rc.emplace_back(i, T.K.col[q]);
  for (auto& e : gp) {
    const int r = T.dim + e.first, c = X.bset[e.second];
    rc.emplace_back(r, c), rc.emplace_back(c, r);
  }
  for (int j = 0; j < X.nM; ++j) rc.emplace_back(T.dim + j, T.dim + j);  // structural zero diagonal
  X.A = pattern_from_pairs(n, n, rc);
  X.kmap.assign(X.A.nnz(), INT32_MIN);
  for (int i = 0; i < T.dim; ++i)
    for (int q = T.K.ptr[i]; q < T.K.ptr[i + 1]; ++q) X.kmap[X.A.find(i, T.K.col[q])] = q;
  for (std::size_t g = 0; g < gp.size(); ++g) {
    const int r = T.dim + gp[g].first, c = X.bset[gp[g].second];
    X.kmap[X.A.find(r, c)] = -2 - (int)g;
    X.kmap[X.A.find(c, r)] = -2 - (int)g;
  }
  for (int& v : X.kmap)
    if (v == INT32_MIN) v = -1000000000;  // structural zero (multiplier diagonal): skipped by the scatter
  // ordering: interior by nested dissection, then B, then the multipliers
  std::vector<int> last(X.bset);
  for (int j = 0; j < X.nM; ++j) last.push_back(T.dim + j);
  std::vector<std::array<int, 2>> ic(T.dof_ic);
  ic.resize(n, {0, 0});
  X.F = analyse(X.A, ic, 16384, 256, 0.15, 16, 48, &last);
  X.root = X.F.nsn - 1;
  if (X.F.sn_col0[X.root] != T.dim - X.nB || X.F.sn_ncol[X.root] != X.nB + X.nM ||
      X.F.sn_nrow[X.root] != X.nB + X.nM) {
    X.why = "root block is not one dense supernode";
    return X;
  }
  X.M = build_front_maps(X.F);
  X.S = build_ascatter(X.F, X.M, X.A, X.kmap.data(), {});
  // drop the structural zeros from the scatter
  AScatter C;
  C.ptr.assign(X.F.nsn + 1, 0);
  for (int k = 0; k < X.F.nsn; ++k) {
    for (int q = X.S.ptr[k]; q < X.S.ptr[k + 1]; ++q)
      if (X.S.kidx[q] != -1000000000) C.kidx.push_back(X.S.kidx[q]), C.fpos.push_back(X.S.fpos[q]);
    C.ptr[k + 1] = (int)C.kidx.size();
  }
  X.S = std::move(C);
  X.ok = true;
  return X;
}

/// G values of a subdomain in the type's pattern order; false if its pattern differs
inline bool dual_sub_values(const DualType& X, const SubType& T, const Subdomain& S, std::vector<int>& lam,
                            std::vector<double>& gval) {
  std::vector<std::tuple<int, int, double>> ent;
  dual_local_mults(S, lam, ent);
  if ((int)lam.size() != X.nM || ent.size() != X.g_j.size()) return false;
  std::vector<int> bpos(T.dim, -1);
  for (int i = 0; i < X.nB; ++i) bpos[X.bset[i]] = i;
  std::vector<std::tuple<int, int, double>> e2;
  for (auto& e : ent) {
    const int b = bpos[std::get<1>(e)];
    if (b < 0) return false;
    e2.emplace_back(std::get<0>(e), b, std::get<2>(e));
  }
  std::sort(e2.begin(), e2.end());
  gval.resize(e2.size());
  for (std::size_t g = 0; g < e2.size(); ++g) {
    if (std::get<0>(e2[g]) != X.g_j[g] || std::get<1>(e2[g]) != X.g_b[g]) return false;
    gval[g] = std::get<2>(e2[g]);
  }
  return true;
}

}  // namespace pf
