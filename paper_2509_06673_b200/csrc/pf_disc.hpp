// pf_disc.hpp — host-side discretisation of the engine: the SX x SY partition
// of the unit square into structured subdomains, their reference numbering,
// constraints, saddle patterns and the mortar multiplier space.
//
// Reference behaviour reproduced (multi-subdomain generalisation of the
// reference's P-below-E pair):
//   * subdomain mesh numbering of mesh.hpp:104-131 (row-major vertices, cells
//     split along the lower-left/upper-right diagonal, edges numbered in
//     discovery order, P2 node = nv + edge);
//   * constraints of assembly.hpp:41-62, symmetric elimination :246-271;
//   * saddle orders P = [u, eta | xi, p], E = [u | xi] (assembly.hpp:338-398);
//   * mortar rows of elements.hpp:234-251, G = +H / -H, constrained columns to
//     H_c (assembly.hpp:401-424), drop rule :106-117.
// Subdomains that share (region, side classes) share one SubType, so the
// symbolic data (patterns, orderings, supernodes, task schedules) exists once
// per type and only numeric values are per subdomain.
#pragma once

#include <map>
#include <thread>
#include <memory>
#include <unordered_map>

#include "pf_common.hpp"

namespace pf {

enum Region { kP = 0, kE = 1 };
enum Side { kLeft = 0, kRight = 1, kBottom = 2, kTop = 3 };

/// Structured cx x cy subdomain topology in reference numbering.
struct Topo {
  int cx = 0, cy = 0, order = 1, nv = 0, ne = 0, nt = 0, nnode = 0;
  std::vector<std::array<int, 3>> tri, tedge;
  std::vector<std::array<int, 2>> edge;
  std::array<std::vector<int>, 4> side_edges;  // ascending along the side
  std::vector<std::array<int, 2>> node_ic;     // half-cell integer coords of u nodes

  int vid(int i, int j) const { return j * (cx + 1) + i; }
  /// local u node list of triangle t in basis order (assembly.hpp:133-144)
  std::array<int, 6> unodes(int t) const {
    return {tri[t][0], tri[t][1], tri[t][2], nv + tedge[t][2], nv + tedge[t][0], nv + tedge[t][1]};
  }
};

inline Topo make_topo(int cx, int cy, int order) {
  Topo T;
  T.cx = cx, T.cy = cy, T.order = order;
  T.nv = (cx + 1) * (cy + 1);
  T.nt = 2 * cx * cy;
  T.tri.reserve(T.nt);
  for (int j = 0; j < cy; ++j)
    for (int i = 0; i < cx; ++i) {
      const int a = T.vid(i, j), b = T.vid(i + 1, j), c = T.vid(i + 1, j + 1), d = T.vid(i, j + 1);
      T.tri.push_back({a, b, c});
      T.tri.push_back({a, c, d});
    }
  std::unordered_map<int64_t, int> ids;
  ids.reserve(std::size_t(3) * T.nt);
  T.tedge.resize(T.nt);
  for (int t = 0; t < T.nt; ++t)
    for (int i = 0; i < 3; ++i) {
      int a = T.tri[t][(i + 1) % 3], b = T.tri[t][(i + 2) % 3];
      if (a > b) std::swap(a, b);
      const int64_t key = int64_t(a) * T.nv + b;
      auto it = ids.find(key);
      if (it == ids.end()) {
        it = ids.emplace(key, (int)T.edge.size()).first;
        T.edge.push_back({a, b});
      }
      T.tedge[t][i] = it->second;
    }
  T.ne = (int)T.edge.size();
  auto eid = [&](int a, int b) { return ids.at(int64_t(std::min(a, b)) * T.nv + std::max(a, b)); };
  for (int i = 0; i < cx; ++i) {
    T.side_edges[kBottom].push_back(eid(T.vid(i, 0), T.vid(i + 1, 0)));
    T.side_edges[kTop].push_back(eid(T.vid(i, cy), T.vid(i + 1, cy)));
  }
  for (int j = 0; j < cy; ++j) {
    T.side_edges[kLeft].push_back(eid(T.vid(0, j), T.vid(0, j + 1)));
    T.side_edges[kRight].push_back(eid(T.vid(cx, j), T.vid(cx, j + 1)));
  }
  T.nnode = T.nv + (order == 2 ? T.ne : 0);
  T.node_ic.resize(T.nnode);
  for (int j = 0; j <= cy; ++j)
    for (int i = 0; i <= cx; ++i) T.node_ic[T.vid(i, j)] = {2 * i, 2 * j};
  if (order == 2)
    for (int e = 0; e < T.ne; ++e) {
      const auto a = T.node_ic[T.edge[e][0]], b = T.node_ic[T.edge[e][1]];
      T.node_ic[T.nv + e] = {(a[0] + b[0]) / 2, (a[1] + b[1]) / 2};
    }
  return T;
}

struct Cons {
  int sidx, node, comp;  // comp -1 = pressure
};

struct SubType {
  int id = 0;
  Region region = kP;
  unsigned outer = 0, pp = 0;  // side bit masks: outer boundary / P|P interface
  std::shared_ptr<const Topo> topo;
  int n_u = 0, n_s = 0, dim = 0, off_eta = -1, off_xi = 0, off_p = -1;
  std::vector<Cons> cons;   // ascending saddle index
  std::vector<int> cpos;    // saddle idx -> constraint position or -1
  bool floating = false;
  std::array<int, 3> fix{-1, -1, -1};
  Csr K;                    // constrained saddle pattern, natural order
  Csr lift;                 // dim x nC pattern (free rows, constrained columns)
  std::vector<int> Bset;    // Dirichlet boundary set: free interface u + free P|P p dofs
  std::vector<std::array<int, 2>> dof_ic;  // half-cell coords per saddle dof
};

struct Subdomain {
  int id = 0, sx = 0, sy = 0, type = 0;
  double x0 = 0, y0 = 0, x1 = 1, y1 = 1;
  // G_s (free columns) and Gc_s (constrained columns), sorted by (lambda, col)
  std::vector<int> g_lam, g_col, gc_lam, gc_col;
  std::vector<double> g_val, gc_val;
};

struct Multiplier {
  int iface, k, comp;  // comp -1 = pressure
};

struct Interface {
  int a, b;
  bool horiz, pp;
};

struct Disc {
  pf_config cfg{};
  Material mat;
  int n = 0, SX = 0, SY = 0, cx = 0, cy = 0;
  std::vector<SubType> types;
  std::vector<Subdomain> subs;
  std::vector<Interface> ifs;
  std::vector<Multiplier> mults;
  int n_lambda = 0, n_lambda_u = 0;
  std::vector<double> kelem;    // injection permeability per global element
  std::vector<uint8_t> srcel;   // injection source indicator per global element
  std::vector<std::array<int, 2>> lambda_ic;  // global half-cell coords per multiplier
  double time(int k) const { return k == mat.N ? mat.T : k * mat.tau; }
};

/// Outer-edge classification of the scenario (model.hpp:260-267, :306-323):
/// returns (displacement component mask, pressure Dirichlet?).
inline std::pair<unsigned, bool> outer_tag(int scenario, Region r, Side side) {
  if (scenario == PF_SCEN_BARRY_MERCER) {
    if (r == kP) return {side == kBottom ? 2u : 1u, true};
    return {side == kTop ? 2u : 1u, false};
  }
  return {3u, r == kP};
}

/// Mortar mass between the P1 multiplier and an order-k trace on an edge of
/// length L (Gauss rule of degree mult+trace+1, elements.hpp:234-251).
inline std::array<std::array<double, 3>, 2> mortar(double L, int trace_order) {
  std::array<std::array<double, 3>, 2> m{};
  std::vector<double> s, w;
  if (trace_order == 1) {
    const double d = 0.5 / std::sqrt(3.0);
    s = {0.5 - d, 0.5 + d};
    w = {0.5, 0.5};
  } else {
    const double d = 0.5 * std::sqrt(3.0 / 5.0);
    s = {0.5 - d, 0.5, 0.5 + d};
    w = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
  }
  for (std::size_t q = 0; q < s.size(); ++q) {
    const double mv[2] = {1 - s[q], s[q]};
    double tv[3];
    if (trace_order == 1) {
      tv[0] = 1 - s[q], tv[1] = s[q], tv[2] = 0;
    } else {
      tv[0] = (1 - s[q]) * (1 - 2 * s[q]), tv[1] = s[q] * (2 * s[q] - 1), tv[2] = 4 * s[q] * (1 - s[q]);
    }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < trace_order + 1; ++j) m[i][j] += w[q] * L * mv[i] * tv[j];
  }
  return m;
}

inline void build_type(SubType& T, const pf_config& cfg) {
  const Topo& tp = *T.topo;
  T.n_u = 2 * tp.nnode;
  T.n_s = tp.nv;
  if (T.region == kP) {
    T.off_eta = T.n_u, T.off_xi = T.n_u + T.n_s, T.off_p = T.n_u + 2 * T.n_s, T.dim = T.n_u + 3 * T.n_s;
  } else {
    T.off_xi = T.n_u, T.dim = T.n_u + T.n_s;
  }
  // constraints (assembly.hpp:41-62)
  std::map<int, Cons> cs;
  for (int side = 0; side < 4; ++side) {
    if (!(T.outer >> side & 1u)) continue;
    const auto [mask, pdir] = outer_tag(cfg.scenario, T.region, (Side)side);
    for (int e : tp.side_edges[side]) {
      int nodes[3] = {tp.edge[e][0], tp.edge[e][1], tp.nv + e};
      const int nn = tp.order == 2 ? 3 : 2;
      for (int c = 0; c < 2; ++c)
        if (mask >> c & 1u)
          for (int q = 0; q < nn; ++q) cs.emplace(2 * nodes[q] + c, Cons{2 * nodes[q] + c, nodes[q], c});
      if (T.region == kP && pdir)
        for (int q = 0; q < 2; ++q) cs.emplace(T.off_p + nodes[q], Cons{T.off_p + nodes[q], nodes[q], -1});
    }
  }
  for (auto& kv : cs) T.cons.push_back(kv.second);
  T.cpos.assign(T.dim, -1);
  for (std::size_t k = 0; k < T.cons.size(); ++k) T.cpos[T.cons[k].sidx] = (int)k;
  T.floating = std::none_of(T.cons.begin(), T.cons.end(), [](const Cons& c) { return c.comp >= 0; });
  if (T.floating) T.fix = {2 * tp.vid(0, 0), 2 * tp.vid(0, 0) + 1, 2 * tp.vid(tp.cx, 0) + 1};
  // saddle pattern from element connectivity
  std::vector<std::pair<int, int>> rc, lc;
  const int nb = tp.order == 2 ? 6 : 3;
  auto add = [&](int r, int c) {
    const bool rcn = T.cpos[r] >= 0, ccn = T.cpos[c] >= 0;
    if (!rcn && !ccn) rc.emplace_back(r, c);
    else if (!rcn && ccn) lc.emplace_back(r, T.cpos[c]);
  };
  rc.reserve(std::size_t(tp.nt) * 600);
  for (int t = 0; t < tp.nt; ++t) {
    const auto un = tp.unodes(t);
    std::vector<int> ud, sd;
    for (int i = 0; i < nb; ++i) ud.push_back(2 * un[i]), ud.push_back(2 * un[i] + 1);
    for (int i = 0; i < 3; ++i) sd.push_back(tp.tri[t][i]);
    for (int r : ud)
      for (int c : ud) add(r, c);
    for (int i : sd)
      for (int c : ud) add(T.off_xi + i, c), add(c, T.off_xi + i);
    for (int i : sd)
      for (int j : sd) {
        if (T.region == kP) {
          add(T.off_eta + i, T.off_eta + j), add(T.off_eta + i, T.off_xi + j), add(T.off_eta + i, T.off_p + j);
          add(T.off_xi + i, T.off_eta + j), add(T.off_xi + i, T.off_xi + j);
          add(T.off_p + i, T.off_eta + j), add(T.off_p + i, T.off_p + j);
        } else {
          add(T.off_xi + i, T.off_xi + j);
        }
      }
  }
  for (const auto& c : T.cons) rc.emplace_back(c.sidx, c.sidx);
  T.K = pattern_from_pairs(T.dim, T.dim, rc);
  T.lift = pattern_from_pairs(T.dim, (int)T.cons.size(), lc);
  // Dirichlet boundary set: trace dofs of interface sides (free), P|P pressure
  std::vector<char> inB(T.dim, 0);
  for (int side = 0; side < 4; ++side) {
    if (T.outer >> side & 1u) continue;
    for (int e : tp.side_edges[side]) {
      int nodes[3] = {tp.edge[e][0], tp.edge[e][1], tp.nv + e};
      for (int q = 0; q < (tp.order == 2 ? 3 : 2); ++q)
        for (int c = 0; c < 2; ++c)
          if (T.cpos[2 * nodes[q] + c] < 0) inB[2 * nodes[q] + c] = 1;
      if (T.pp >> side & 1u)
        for (int q = 0; q < 2; ++q)
          if (T.cpos[T.off_p + nodes[q]] < 0) inB[T.off_p + nodes[q]] = 1;
    }
  }
  for (int i = 0; i < T.dim; ++i)
    if (inB[i]) T.Bset.push_back(i);
  T.dof_ic.resize(T.dim);
  for (int nd = 0; nd < tp.nnode; ++nd) T.dof_ic[2 * nd] = T.dof_ic[2 * nd + 1] = tp.node_ic[nd];
  for (int v = 0; v < tp.nv; ++v) {
    T.dof_ic[T.off_xi + v] = tp.node_ic[v];
    if (T.region == kP) T.dof_ic[T.off_eta + v] = T.dof_ic[T.off_p + v] = tp.node_ic[v];
  }
}

inline Disc build_disc(const pf_config& cfg, const double* k_override) {
  Disc D;
  D.cfg = cfg;
  if (cfg.order != 1 && cfg.order != 2) fail(kInvalid, "fe_order must be 1 or 2");
  if (cfg.scenario < 0 || cfg.scenario > 3) fail(kInvalid, "unknown scenario id");
  if (cfg.precond < 0 || cfg.precond > 4) fail(kInvalid, "unknown preconditioner id");
  if (cfg.krylov < 0 || cfg.krylov > 4) fail(kInvalid, "unknown krylov id");
  if (cfg.SX < 1 || cfg.SY < 2 || cfg.SY % 2)
    fail(kInvalid, "partition needs SX >= 1 and an even SY >= 2 (P below y=1/2, E above)");
  if (cfg.mesh_n < 1 || cfg.mesh_n % cfg.SX || cfg.mesh_n % cfg.SY)
    fail(kInvalid, "mesh_n must be divisible by SX and SY");
  if (!(cfg.tol > 0)) fail(kNotConverged, "feti_pcg: tolerance must be positive");
  D.mat = make_material(cfg);
  D.n = cfg.mesh_n, D.SX = cfg.SX, D.SY = cfg.SY;
  D.cx = D.n / D.SX, D.cy = D.n / D.SY;
  auto topo = std::make_shared<const Topo>(make_topo(D.cx, D.cy, cfg.order));
  if (cfg.scenario == PF_SCEN_INJECTION) {
    if (k_override)
      D.kelem.assign(k_override, k_override + std::size_t(2) * D.n * D.n);
    else
      D.kelem = injection_permeability(D.n, cfg.seed, cfg.logk_mean, cfg.logk_sd);
    D.srcel.assign(std::size_t(2) * D.n * D.n, 0);
    const double h = 1.0 / D.n;
    for (int J = 0; J < D.n; ++J)
      for (int I = 0; I < D.n; ++I)
        for (int k = 0; k < 2; ++k) {
          // centroid ((p0 + p1) + p2) / 3 of (a,b,c) resp. (a,c,d)
          const double ax = I * h, ay = J * h, bx = (I + 1) * h, by = J * h;
          const double cxx = (I + 1) * h, cyy = (J + 1) * h, dx0 = I * h, dy0 = (J + 1) * h;
          const double gx = k == 0 ? ((ax + bx) + cxx) * (1.0 / 3.0) : ((ax + cxx) + dx0) * (1.0 / 3.0);
          const double gy = k == 0 ? ((ay + by) + cyy) * (1.0 / 3.0) : ((ay + cyy) + dy0) * (1.0 / 3.0);
          const double dx = gx - 0.5, dy = gy - 0.25;
          D.srcel[2 * (J * D.n + I) + k] = std::sqrt(dx * dx + dy * dy) <= 0.02;
        }
  }
  // subdomains and types
  std::map<std::array<unsigned, 3>, int> type_of;
  D.subs.resize(D.SX * D.SY);
  for (int sy = 0; sy < D.SY; ++sy)
    for (int sx = 0; sx < D.SX; ++sx) {
      Subdomain& S = D.subs[sy * D.SX + sx];
      S.id = sy * D.SX + sx, S.sx = sx, S.sy = sy;
      S.x0 = double(sx * D.cx) / D.n, S.y0 = double(sy * D.cy) / D.n;
      S.x1 = double((sx + 1) * D.cx) / D.n, S.y1 = double((sy + 1) * D.cy) / D.n;
      const Region reg = 2 * (sy + 1) <= D.SY ? kP : kE;
      unsigned outer = 0, pp = 0;
      if (sx == 0) outer |= 1u << kLeft;
      if (sx == D.SX - 1) outer |= 1u << kRight;
      if (sy == 0) outer |= 1u << kBottom;
      if (sy == D.SY - 1) outer |= 1u << kTop;
      if (reg == kP) {
        auto isP = [&](int y) { return 2 * (y + 1) <= D.SY; };
        if (sx > 0) pp |= 1u << kLeft;
        if (sx < D.SX - 1) pp |= 1u << kRight;
        if (sy > 0) pp |= 1u << kBottom;
        if (sy < D.SY - 1 && isP(sy + 1)) pp |= 1u << kTop;
      }
      const std::array<unsigned, 3> key{(unsigned)reg, outer, pp};
      auto it = type_of.find(key);
      if (it == type_of.end()) {
        SubType T;
        T.id = (int)D.types.size(), T.region = reg, T.outer = outer, T.pp = pp, T.topo = topo;
        it = type_of.emplace(key, T.id).first;
        D.types.push_back(std::move(T));
      }
      S.type = it->second;
    }
  // the per-type patterns are independent: one thread per type
  {
    std::vector<std::thread> th;
    for (auto& T : D.types) th.emplace_back([&T, &cfg] { build_type(T, cfg); });
    for (auto& t : th) t.join();
  }
  // interfaces: per subdomain top then right (same enumeration as the oracle)
  for (int sy = 0; sy < D.SY; ++sy)
    for (int sx = 0; sx < D.SX; ++sx) {
      const int s = sy * D.SX + sx;
      if (sy + 1 < D.SY)
        D.ifs.push_back({s, s + D.SX, true,
                         D.types[D.subs[s].type].region == kP && D.types[D.subs[s + D.SX].type].region == kP});
      if (sx + 1 < D.SX)
        D.ifs.push_back({s, s + 1, false,
                         D.types[D.subs[s].type].region == kP && D.types[D.subs[s + 1].type].region == kP});
    }
  const Topo& tp = *topo;
  auto seg_vertex = [&](const Interface& I, int side_ab, int k) {  // vertex id on side a(0)/b(1)
    if (I.horiz) return side_ab == 0 ? tp.vid(k, tp.cy) : tp.vid(k, 0);
    return side_ab == 0 ? tp.vid(tp.cx, k) : tp.vid(0, k);
  };
  auto seg_edges = [&](const Interface& I, int side_ab) -> const std::vector<int>& {
    if (I.horiz) return tp.side_edges[side_ab == 0 ? kTop : kBottom];
    return tp.side_edges[side_ab == 0 ? kRight : kLeft];
  };
  // multipliers (u on every interface, then p on P|P)
  std::map<std::array<int, 3>, int> mindex;
  for (int pass = 0; pass < 2; ++pass) {
    for (int f = 0; f < (int)D.ifs.size(); ++f) {
      const Interface& I = D.ifs[f];
      if (pass == 1 && !I.pp) continue;
      const SubType &Ta = D.types[D.subs[I.a].type], &Tb = D.types[D.subs[I.b].type];
      const int nk = (I.horiz ? tp.cx : tp.cy) + 1;
      const bool cross_row = !I.horiz && D.subs[I.a].sy >= 1;
      for (int k = 0; k < nk; ++k) {
        const int va = seg_vertex(I, 0, k), vb = seg_vertex(I, 1, k);
        const bool cross = cross_row && k == 0;
        if (pass == 0) {
          for (int c = 0; c < 2; ++c) {
            if (Ta.cpos[2 * va + c] >= 0 && Tb.cpos[2 * vb + c] >= 0) continue;
            if (cfg.order == 1 && cross) continue;
            mindex[{f, k, c}] = (int)D.mults.size();
            D.mults.push_back({f, k, c});
          }
        } else {
          if (Ta.cpos[Ta.off_p + va] >= 0 && Tb.cpos[Tb.off_p + vb] >= 0) continue;
          if (cross) continue;
          mindex[{f, k, -1}] = (int)D.mults.size();
          D.mults.push_back({f, k, -1});
        }
      }
    }
    if (pass == 0) D.n_lambda_u = (int)D.mults.size();
  }
  D.n_lambda = (int)D.mults.size();
  D.lambda_ic.resize(D.n_lambda);
  for (int i = 0; i < D.n_lambda; ++i) {
    const Multiplier& m = D.mults[i];
    const Interface& I = D.ifs[m.iface];
    const Subdomain& Sa = D.subs[I.a];
    const int gi = I.horiz ? Sa.sx * D.cx + m.k : (Sa.sx + 1) * D.cx;
    const int gj = I.horiz ? (Sa.sy + 1) * D.cy : Sa.sy * D.cy + m.k;
    D.lambda_ic[i] = {2 * gi, 2 * gj};
  }
  // G / Gc entries with REF accumulation order (edge by edge)
  std::vector<std::map<std::pair<int, int>, double>> G(D.subs.size()), Gc(D.subs.size());
  // per subdomain (threads), its interfaces in ascending order: every entry
  // accumulates its contributions in the same order as an interface-major loop
  std::vector<std::vector<std::pair<int, int>>> ifs_of(D.subs.size());
  for (int f = 0; f < (int)D.ifs.size(); ++f)
    ifs_of[D.ifs[f].a].emplace_back(f, 0), ifs_of[D.ifs[f].b].emplace_back(f, 1);
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto build_g = [&](int s_begin, int s_step) {
  for (int s_ = s_begin; s_ < (int)D.subs.size(); s_ += s_step)
  for (const auto& fs : ifs_of[s_]) {
    const int f = fs.first;
    const Interface& I = D.ifs[f];
    const int nseg = I.horiz ? tp.cx : tp.cy;
    for (int side = fs.second; side == fs.second; ++side) {
      const Subdomain& S = D.subs[side == 0 ? I.a : I.b];
      const SubType& T = D.types[S.type];
      const double sign = side == 0 ? 1.0 : -1.0;
      const double hx = (S.x1 - S.x0) / tp.cx, hy = (S.y1 - S.y0) / tp.cy;
      const Subdomain& Sa = D.subs[I.a];
      const double hxa = (Sa.x1 - Sa.x0) / tp.cx, hya = (Sa.y1 - Sa.y0) / tp.cy;
      (void)hx, (void)hy;
      for (int j = 0; j < nseg; ++j) {
        // geometry from side a's vertex coordinates (REF uses the P-side edge, assembly.hpp:212)
        const int va0 = seg_vertex(I, 0, j), va1 = seg_vertex(I, 0, j + 1);
        const double ax = Sa.x0 + (va0 % (tp.cx + 1)) * hxa, ay = Sa.y0 + (va0 / (tp.cx + 1)) * hya;
        const double bx = Sa.x0 + (va1 % (tp.cx + 1)) * hxa, by = Sa.y0 + (va1 / (tp.cx + 1)) * hya;
        const double L = std::sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay));
        const auto H = mortar(L, cfg.order);
        const auto Hp = mortar(L, 1);
        const int e = seg_edges(I, side)[j];
        const int nodes[3] = {seg_vertex(I, side, j), seg_vertex(I, side, j + 1), tp.nv + e};
        const int nq = cfg.order == 2 ? 3 : 2;
        for (int i = 0; i < 2; ++i) {
          for (int c = 0; c < 2; ++c) {
            auto it = mindex.find({f, j + i, c});
            if (it == mindex.end()) continue;
            for (int q = 0; q < nq; ++q) {
              const int col = 2 * nodes[q] + c;
              if (T.cpos[col] >= 0)
                Gc[S.id][{it->second, T.cpos[col]}] += sign * H[i][q];
              else
                G[S.id][{it->second, col}] += sign * H[i][q];
            }
          }
          if (I.pp) {
            auto it = mindex.find({f, j + i, -1});
            if (it == mindex.end()) continue;
            for (int q = 0; q < 2; ++q) {
              const int col = T.off_p + nodes[q];
              if (T.cpos[col] >= 0)
                Gc[S.id][{it->second, T.cpos[col]}] += sign * Hp[i][q];
              else
                G[S.id][{it->second, col}] += sign * Hp[i][q];
            }
          }
        }
      }
    }
  }
  };
  {
    std::vector<std::thread> th;
    for (int k = 0; k < nth; ++k) th.emplace_back(build_g, k, nth);
    for (auto& t : th) t.join();
  }
  for (auto& S : D.subs) {
    for (auto& kv : G[S.id]) S.g_lam.push_back(kv.first.first), S.g_col.push_back(kv.first.second), S.g_val.push_back(kv.second);
    for (auto& kv : Gc[S.id]) S.gc_lam.push_back(kv.first.first), S.gc_col.push_back(kv.first.second), S.gc_val.push_back(kv.second);
  }
  return D;
}

}  // namespace pf
