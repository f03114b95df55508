// pf_iface.hpp — symbolic analysis of the sparse direct interface solve: a
// nested dissection of the multiplier space over the subdomain grid.
//
// The interface operator F = sum_s B_s F_s B_s^T is assembled like a finite
// element matrix whose "elements" are the subdomains (dense F_s on the
// subdomain's multipliers) and whose "nodes" are the multipliers; a multiplier
// lies on one interface (a, b) and so couples exactly two subdomains.  A
// rectangle R of subdomains is bisected along its longer side into R1 and R2:
//   sep(R)  = multipliers with both subdomains in R but on different halves
//             (fully summed once R1 and R2 are condensed),
//   bdry(R) = multipliers with exactly one subdomain in R.
// Front(R) = [sep(R) | bdry(R)] receives the Schur complements of R1 and R2 on
// bdry(R1) and bdry(R2) (a single subdomain's is its F_s), eliminates sep(R)
// and hands its own Schur complement on bdry(R) to its parent (multifrontal
// extend-add).  The reference has no counterpart: its MonolithicSolver
// (feti.hpp:313-440) factors the whole coupled system with SparseLU; this is
// the same exact condensation carried one level further, onto the multipliers.
#pragma once

#include <algorithm>
#include <vector>

#include "pf_disc.hpp"

namespace pf {

struct IfaceFront {
  static constexpr int kNone = -(1 << 30);
  int nsep = 0, nbdry = 0, depth = 0;
  int child[2] = {kNone, kNone};    // >= 0: front; kNone: nothing; else leaf subdomain -(s + 1)
  std::vector<int> idx;             // global multipliers: separator first, then boundary
  std::vector<unsigned char> side;  // per boundary entry: 0 = the interface's subdomain a lies in R, 1 = b
  int m() const { return nsep + nbdry; }
};

struct IfaceTree {
  std::vector<IfaceFront> fronts;  // post-order: children before parents; the root is last
  int ndepth = 0;
  long long factor_values = 0;     // sum over fronts of nsep * (nsep + 2 nbdry)
};

namespace iface_detail {
struct Rect {
  int x0, x1, y0, y1;
  bool has(const Subdomain& S) const { return S.sx >= x0 && S.sx < x1 && S.sy >= y0 && S.sy < y1; }
};

inline int build(const Disc& D, const std::vector<int>& grid, IfaceTree& T, Rect R, const std::vector<int>& touch,
                 int depth) {
  const int w = R.x1 - R.x0, h = R.y1 - R.y0;
  if (w * h == 1) return -(grid[R.x0 + R.y0 * D.SX] + 1);
  Rect R1 = R, R2 = R;
  if (w >= h) R1.x1 = R2.x0 = R.x0 + w / 2;
  else R1.y1 = R2.y0 = R.y0 + h / 2;
  IfaceFront F;
  F.depth = depth;
  std::vector<int> t1, t2, sep, bd;
  std::vector<unsigned char> bside;
  for (int g : touch) {
    const Interface& I = D.ifs[D.mults[g].iface];
    const Subdomain &A = D.subs[I.a], &B = D.subs[I.b];
    const bool ina = R.has(A), inb = R.has(B);
    if (ina && inb) {
      const bool a1 = R1.has(A), b1 = R1.has(B);
      if (a1 && b1) t1.push_back(g);
      else if (!a1 && !b1) t2.push_back(g);
      else sep.push_back(g), t1.push_back(g), t2.push_back(g);
    } else {
      bd.push_back(g), bside.push_back(ina ? 0 : 1);
      (R1.has(ina ? A : B) ? t1 : t2).push_back(g);
    }
  }
  F.nsep = (int)sep.size(), F.nbdry = (int)bd.size();
  F.idx = sep, F.idx.insert(F.idx.end(), bd.begin(), bd.end());
  F.side = bside;
  F.child[0] = build(D, grid, T, R1, t1, depth + 1);
  F.child[1] = build(D, grid, T, R2, t2, depth + 1);
  T.ndepth = std::max(T.ndepth, depth + 1);
  T.factor_values += (long long)F.nsep * (F.nsep + 2LL * F.nbdry);
  T.fronts.push_back(std::move(F));
  return (int)T.fronts.size() - 1;
}
}  // namespace iface_detail

/// Nested dissection of the multipliers over the SX x SY subdomain grid.
inline IfaceTree build_iface_tree(const Disc& D) {
  IfaceTree T;
  std::vector<int> grid((std::size_t)D.SX * D.SY, -1);
  for (const Subdomain& S : D.subs) grid[S.sx + S.sy * D.SX] = S.id;
  std::vector<int> all(D.n_lambda);
  for (int g = 0; g < D.n_lambda; ++g) all[g] = g;
  if (D.SX * D.SY > 1) iface_detail::build(D, grid, T, iface_detail::Rect{0, D.SX, 0, D.SY}, all, 0);
  return T;
}

}  // namespace pf
