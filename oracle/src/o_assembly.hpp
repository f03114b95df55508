// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// o_assembly.hpp — restatement of assembly.hpp generalised from the
// reference's two subdomains (P below E) to an SX x SY partition (SURVEY
// App. C D1-D5):
//   constraints (assembly.hpp:41-76), subdomain blocks (:148-197), interface
//   mortar (:201-235), symmetric elimination + lifting (:240-276), saddle
//   assembly in the [u, eta | xi, p] / [u | xi] orders with the block signs of
//   :363-373 and :389-393, signed coupling G with constrained columns moved to
//   H_c (:401-424), per-step loads and right-hand sides (:430-579).
// Multi-subdomain rules (identical in the product):
//   * interfaces enumerated per subdomain s = sy*SX+sx: top (s|s+SX) then
//     right (s|s+1); sign +1 for the lower/left side, -1 for the other;
//   * u multipliers: P1 vector on the segment vertices (ascending along the
//     segment, node-major / component-minor), all interfaces first; then
//     scalar P1 p multipliers on P|P interfaces;
//   * a multiplier is dropped when both sides' trace dofs are essential
//     (assembly.hpp:106-117); for P1 traces (order-1 u, and always p) the
//     bottom multiplier of a vertical interface whose bottom vertex is an
//     interior cross point is dropped (P1 mortar rows are M * pointwise jumps,
//     so the four cross-point rows have rank 3);
//   * floating subdomains (no essential u) get fixing dofs (vertex 0 both
//     components, vertex nx component 1) and rigid modes (1,0),(0,1),
//     (-(y-yc), x-xc).
#pragma once

#include <map>
#include <set>
#include <tuple>

#include "o_elements.hpp"
#include "o_model.hpp"

namespace oracle {

struct Config {
  std::string scenario = "mms-t";
  int mesh_n = 32, SX = 1, SY = 2, order = 1;
  double E = 1.0, nu = 0.3, alpha = 1.0, c0 = 1e-3, kperm = 1.0, mu_f = 1.0;
  double dt = 1e-2;
  int steps = 5;
  MuConv conv = MuConv::paper;
  uint64_t seed = 20240901ull;
  double logk_mean = -2.0, logk_sd = 1.0;
  std::string precond = "dirichlet";  // identity | generalized | dirichlet
  std::string krylov = "auto";        // auto | pcg | minres
  double tol = 1e-10;
  int max_iter = 500;
  bool warm = true;
  int threads = 0;  // 0 = hardware concurrency
};

struct Cons {
  int sidx;  // saddle index
  bool is_u;
  int comp;
  V2 xy;
};

struct Sub {
  int id = 0, sx = 0, sy = 0;
  Region region = Region::P;
  Mesh mesh;
  DofMap u, s;
  int n_u = 0, n_s = 0, dim = 0, off_u = 0, off_eta = 0, off_xi = 0, off_p = 0;
  std::vector<int> gelem;   // global element id per local triangle
  Csr A, B, R, Af;          // raw blocks
  Csr K;                    // constrained saddle (identity rows at constraints)
  Csr lift;                 // dim x nC, original columns at constraints, free rows
  std::vector<Cons> cons;   // ordered like ascending saddle index
  std::vector<int> cpos;    // saddle idx -> constraint position or -1
  Csr G, Gc;                // n_lambda x dim (signed, free cols); n_lambda x nC (signed)
  bool floating = false;
  std::vector<int> fix;     // fixing saddle dofs (floating only)
  Dense Rk;                 // dim x 3 rigid modes (floating only)
  std::vector<int> Bu, Bp;  // Dirichlet-preconditioner boundary sets (saddle idx)
};

struct Iface {
  int a = 0, b = 0;
  bool horiz = true, pp = false;
  std::vector<int> va, vb, ea, eb;  // vertices / edges along the segment, ascending
};

struct Mult {
  int iface, k, comp;  // comp -1 = pressure
};

struct Disc {
  Config cfg;
  Params par;
  Scenario sc;
  double T = 0, tau = 0;
  int N = 0;
  std::vector<Sub> subs;
  std::vector<Iface> ifs;
  std::vector<Mult> mults;
  int n_lambda = 0, n_lambda_u = 0;
  std::vector<double> kelem;   // per global element permeability (injection)
  std::vector<char> src_elem;  // per global element source indicator (injection)
  double time(int n) const { return n == N ? T : n * tau; }
};

namespace detail {

inline std::vector<int> local_u_nodes(const Mesh& m, int t, int order) {
  std::vector<int> n = {m.tri[t][0], m.tri[t][1], m.tri[t][2]};
  if (order == 2) {
    n.push_back(m.nv() + m.tedge[t][2]);
    n.push_back(m.nv() + m.tedge[t][0]);
    n.push_back(m.nv() + m.tedge[t][1]);
  }
  return n;
}

inline void add_block(std::vector<Trip>& ts, const Csr& M, int ro, int co, double s, bool tr = false) {
  for (int i = 0; i < M.nr; ++i)
    for (int q = M.ptr[i]; q < M.ptr[i + 1]; ++q)
      if (tr)
        ts.push_back({ro + M.col[q], co + i, s * M.val[q]});
      else
        ts.push_back({ro + i, co + M.col[q], s * M.val[q]});
}

}  // namespace detail

inline void assemble_blocks(Sub& S, const Disc& D) {
  const Mesh& m = S.mesh;
  const double mu = S.region == Region::P ? D.par.mu_P : D.par.mu_E;
  std::vector<Trip> ta, tb, tr, tf;
  for (int t = 0; t < m.nt(); ++t) {
    const auto c = m.coords(t);
    const auto un = detail::local_u_nodes(m, t, S.u.order);
    const auto& sn = m.tri[t];
    const int nb = (int)un.size();
    const Dense la = local_elastic(c, mu, S.u.order);
    for (int i = 0; i < nb; ++i)
      for (int ci = 0; ci < 2; ++ci)
        for (int j = 0; j < nb; ++j)
          for (int cj = 0; cj < 2; ++cj)
            ta.push_back({S.u.dof(un[i], ci), S.u.dof(un[j], cj), la(2 * i + ci, 2 * j + cj)});
    const Dense lb = local_div(c, S.u.order);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < nb; ++j)
        for (int cj = 0; cj < 2; ++cj) tb.push_back({sn[i], S.u.dof(un[j], cj), lb(i, 2 * j + cj)});
    const Dense lr = local_mass(c);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) tr.push_back({sn[i], sn[j], lr(i, j)});
    if (S.region == Region::P) {
      double k00 = D.par.K00, k01 = D.par.K01, k11 = D.par.K11;
      if (!D.kelem.empty()) k00 = k11 = D.kelem[S.gelem[t]], k01 = 0.0;
      const Dense lf = local_diffusion(c, k00, k01, k11, D.par.mu_f);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) tf.push_back({sn[i], sn[j], lf(i, j)});
    }
  }
  S.A = Csr::from_trips(S.u.ndof, S.u.ndof, ta);
  S.B = Csr::from_trips(S.s.ndof, S.u.ndof, tb);
  S.R = Csr::from_trips(S.s.ndof, S.s.ndof, tr);
  if (S.region == Region::P) S.Af = Csr::from_trips(S.s.ndof, S.s.ndof, tf);
}

/// Symmetric elimination (assembly.hpp:246-271).
inline void eliminate(Sub& S, const Csr& M) {
  std::vector<Trip> tm, tl;
  for (int i = 0; i < M.nr; ++i)
    for (int q = M.ptr[i]; q < M.ptr[i + 1]; ++q) {
      const int j = M.col[q];
      const bool rc = S.cpos[i] >= 0, cc = S.cpos[j] >= 0;
      if (!rc && !cc)
        tm.push_back({i, j, M.val[q]});
      else if (!rc && cc)
        tl.push_back({i, S.cpos[j], M.val[q]});
    }
  for (const auto& c : S.cons) tm.push_back({c.sidx, c.sidx, 1.0});
  S.K = Csr::from_trips(M.nr, M.nc, tm);
  S.lift = Csr::from_trips(M.nr, (int)S.cons.size(), tl);
}

inline Disc build_discretization(const Config& cfg) {
  Disc D;
  D.cfg = cfg;
  if (cfg.order != 1 && cfg.order != 2) throw ConfigError("fe_order must be 1 or 2");
  if (cfg.SX < 1 || cfg.SY < 2 || cfg.SY % 2 != 0)
    throw ConfigError("partition needs SX >= 1 and an even SY >= 2 (P below y=1/2, E above)");
  if (cfg.mesh_n % cfg.SX != 0 || cfg.mesh_n % cfg.SY != 0)
    throw ConfigError("mesh_n must be divisible by SX and SY");
  if (!(cfg.dt > 0) || cfg.steps < 1) throw ConfigError("need dt > 0 and steps >= 1");
  D.par = make_params(cfg.E, cfg.nu, cfg.E, cfg.nu, cfg.alpha, cfg.c0, cfg.kperm, cfg.mu_f, cfg.conv);
  D.sc = scenario_by_name(cfg.scenario, D.par);
  // time grid (timeloop.hpp:15-33): N = max(1, llround(T/dt)), tau = T/N
  D.T = cfg.dt * cfg.steps;
  D.N = std::max(1, (int)std::llround(D.T / cfg.dt));
  D.tau = D.T / D.N;
  const int n = cfg.mesh_n, SX = cfg.SX, SY = cfg.SY, cx = n / SX, cy = n / SY;
  if (D.sc.per_element) {
    D.kelem = lognormal_permeability(n, cfg.seed, cfg.logk_mean, cfg.logk_sd);
    D.src_elem.assign(std::size_t(2) * n * n, 0);
    const double h = 1.0 / n;
    for (int J = 0; J < n; ++J)
      for (int I = 0; I < n; ++I) {
        const V2 a(I * h, J * h), b((I + 1) * h, J * h), c((I + 1) * h, (J + 1) * h), d(I * h, (J + 1) * h);
        const V2 c0 = (a + b + c) * (1.0 / 3.0), c1 = (a + c + d) * (1.0 / 3.0);
        const V2 s(D.sc.src_x, D.sc.src_y);
        D.src_elem[2 * (J * n + I)] = (c0 - s).norm() <= D.sc.src_r;
        D.src_elem[2 * (J * n + I) + 1] = (c1 - s).norm() <= D.sc.src_r;
      }
  }
  // subdomains
  D.subs.resize(SX * SY);
  for (int sy = 0; sy < SY; ++sy)
    for (int sx = 0; sx < SX; ++sx) {
      Sub& S = D.subs[sy * SX + sx];
      S.id = sy * SX + sx;
      S.sx = sx;
      S.sy = sy;
      S.region = (2 * (sy + 1) <= SY) ? Region::P : Region::E;
      const Rect r{double(sx * cx) / n, double(sy * cy) / n, double((sx + 1) * cx) / n,
                   double((sy + 1) * cy) / n};
      S.mesh = build_subdomain_mesh(S.region, r, cx, cy);
      const Scenario& sc = D.sc;
      const Region reg = S.region;
      S.mesh = tag_boundary_facets(S.mesh, [&sc, reg](const V2& m) -> std::optional<Tag> {
        const bool outer = near(m.x, 0.0) || near(m.x, 1.0) || near(m.y, 0.0) || near(m.y, 1.0);
        if (!outer) return Tag::iface();
        return sc.outer_tag(reg, m);
      });
      S.gelem.resize(S.mesh.nt());
      for (int t = 0; t < S.mesh.nt(); ++t) {
        const int cell = t / 2, i = cell % cx, j = cell / cx;
        S.gelem[t] = 2 * ((sy * cy + j) * n + (sx * cx + i)) + (t % 2);
      }
      S.u = make_dof_map(S.mesh, Field::disp, cfg.order);
      S.s = make_dof_map(S.mesh, Field::xi, 1);
      S.n_u = S.u.ndof;
      S.n_s = S.s.ndof;
      S.off_u = 0;
      if (S.region == Region::P) {
        S.off_eta = S.n_u;
        S.off_xi = S.n_u + S.n_s;
        S.off_p = S.n_u + 2 * S.n_s;
        S.dim = S.n_u + 3 * S.n_s;
      } else {
        S.off_xi = S.n_u;
        S.dim = S.n_u + S.n_s;
        S.off_eta = S.off_p = -1;
      }
      // constraints (assembly.hpp:41-62), ascending saddle index
      std::map<int, Cons> cs;
      for (const auto& be : S.mesh.bnd) {
        if (be.tag.interface_edge) continue;
        const int e = be.edge;
        std::vector<int> nodes = {S.mesh.edge[e][0], S.mesh.edge[e][1]};
        if (cfg.order == 2) nodes.push_back(S.mesh.nv() + e);
        for (int c = 0; c < 2; ++c) {
          if (!be.tag.essential(c)) continue;
          for (int nd : nodes) cs.emplace(S.off_u + S.u.dof(nd, c), Cons{S.off_u + S.u.dof(nd, c), true, c, S.u.xy[nd]});
        }
        if (S.region == Region::P && be.tag.pressure == PTag::dirichlet)
          for (int v : {S.mesh.edge[e][0], S.mesh.edge[e][1]})
            cs.emplace(S.off_p + v, Cons{S.off_p + v, false, 0, S.s.xy[v]});
      }
      for (auto& kv : cs) S.cons.push_back(kv.second);
      S.cpos.assign(S.dim, -1);
      for (std::size_t k = 0; k < S.cons.size(); ++k) S.cpos[S.cons[k].sidx] = (int)k;
      S.floating = std::none_of(S.cons.begin(), S.cons.end(), [](const Cons& c) { return c.is_u; });
      assemble_blocks(S, D);
      // saddle (assembly.hpp:348-398)
      std::vector<Trip> ts;
      const Params& P = D.par;
      if (S.region == Region::P) {
        detail::add_block(ts, S.A, S.off_u, S.off_u, 1.0);
        detail::add_block(ts, S.R, S.off_eta, S.off_eta, P.k2);
        detail::add_block(ts, S.B, S.off_u, S.off_xi, 1.0, true);
        detail::add_block(ts, S.R, S.off_eta, S.off_xi, P.k1);
        detail::add_block(ts, S.R, S.off_eta, S.off_p, -1.0);
        detail::add_block(ts, S.B, S.off_xi, S.off_u, 1.0);
        detail::add_block(ts, S.R, S.off_xi, S.off_eta, P.k1);
        detail::add_block(ts, S.R, S.off_xi, S.off_xi, -P.k3);
        detail::add_block(ts, S.R, S.off_p, S.off_eta, -1.0);
        detail::add_block(ts, S.Af, S.off_p, S.off_p, -D.tau);
      } else {
        detail::add_block(ts, S.A, S.off_u, S.off_u, 1.0);
        detail::add_block(ts, S.B, S.off_u, S.off_xi, 1.0, true);
        detail::add_block(ts, S.B, S.off_xi, S.off_u, 1.0);
        detail::add_block(ts, S.R, S.off_xi, S.off_xi, -1.0 / P.lam_E);
      }
      eliminate(S, Csr::from_trips(S.dim, S.dim, ts));
      if (S.floating) {
        const int v0 = 0, v1 = S.mesh.nx;
        S.fix = {S.off_u + S.u.dof(v0, 0), S.off_u + S.u.dof(v0, 1), S.off_u + S.u.dof(v1, 1)};
        const V2 ctr((r.x0 + r.x1) * 0.5, (r.y0 + r.y1) * 0.5);
        S.Rk = Dense(S.dim, 3);
        for (int nd = 0; nd < S.u.nnode; ++nd) {
          const V2 x = S.u.xy[nd];
          S.Rk(S.off_u + S.u.dof(nd, 0), 0) = 1.0;
          S.Rk(S.off_u + S.u.dof(nd, 1), 1) = 1.0;
          S.Rk(S.off_u + S.u.dof(nd, 0), 2) = -(x.y - ctr.y);
          S.Rk(S.off_u + S.u.dof(nd, 1), 2) = x.x - ctr.x;
        }
      }
    }
  // interfaces
  auto seg = [&](const Sub& S, bool horiz, bool top_or_right) {
    // interface edges of S lying on the requested side, sorted along the segment
    std::vector<std::pair<double, int>> es;
    const Rect& r = S.mesh.rect;
    for (const auto& be : S.mesh.bnd) {
      if (!be.tag.interface_edge) continue;
      const V2 m = S.mesh.mid(be.edge);
      const bool on = horiz ? near(m.y, top_or_right ? r.y1 : r.y0) : near(m.x, top_or_right ? r.x1 : r.x0);
      if (on) es.emplace_back(horiz ? m.x : m.y, be.edge);
    }
    std::sort(es.begin(), es.end());
    std::vector<int> edges, verts;
    for (auto& p : es) edges.push_back(p.second);
    for (std::size_t j = 0; j < edges.size(); ++j) {
      int a = S.mesh.edge[edges[j]][0], b = S.mesh.edge[edges[j]][1];
      const double ca = horiz ? S.mesh.vtx[a].x : S.mesh.vtx[a].y;
      const double cb = horiz ? S.mesh.vtx[b].x : S.mesh.vtx[b].y;
      if (ca > cb) std::swap(a, b);
      if (j == 0) verts.push_back(a);
      verts.push_back(b);
    }
    return std::make_pair(edges, verts);
  };
  for (int sy = 0; sy < SY; ++sy)
    for (int sx = 0; sx < SX; ++sx) {
      const int s = sy * SX + sx;
      for (int dir = 0; dir < 2; ++dir) {
        const bool horiz = dir == 0;
        if (horiz && sy + 1 >= SY) continue;
        if (!horiz && sx + 1 >= SX) continue;
        Iface I;
        I.a = s;
        I.b = horiz ? s + SX : s + 1;
        I.horiz = horiz;
        I.pp = D.subs[I.a].region == Region::P && D.subs[I.b].region == Region::P;
        auto A = seg(D.subs[I.a], horiz, true), B = seg(D.subs[I.b], horiz, false);
        I.ea = A.first, I.va = A.second, I.eb = B.first, I.vb = B.second;
        if (I.va.size() != I.vb.size() || I.va.empty())
          throw NonConformingInterfaceError("interface trace counts differ");
        for (std::size_t k = 0; k < I.va.size(); ++k)
          if ((D.subs[I.a].mesh.vtx[I.va[k]] - D.subs[I.b].mesh.vtx[I.vb[k]]).linf() > kGeomTol)
            throw NonConformingInterfaceError("interface node mismatch");
        D.ifs.push_back(I);
      }
    }
  // multipliers: u on all interfaces, then p on P|P
  auto constrained = [](const Sub& S, int sidx) { return S.cpos[sidx] >= 0; };
  for (int pass = 0; pass < 2; ++pass) {
    for (int f = 0; f < (int)D.ifs.size(); ++f) {
      const Iface& I = D.ifs[f];
      const Sub &Sa = D.subs[I.a], &Sb = D.subs[I.b];
      if (pass == 1 && !I.pp) continue;
      for (int k = 0; k < (int)I.va.size(); ++k) {
        const bool cross = !I.horiz && Sa.sy >= 1 && k == 0;  // interior cross point below
        if (pass == 0) {
          for (int c = 0; c < 2; ++c) {
            const bool both = constrained(Sa, Sa.off_u + Sa.u.dof(I.va[k], c)) &&
                              constrained(Sb, Sb.off_u + Sb.u.dof(I.vb[k], c));
            if (both || (cfg.order == 1 && cross)) continue;
            D.mults.push_back({f, k, c});
          }
        } else {
          const bool both = constrained(Sa, Sa.off_p + I.va[k]) && constrained(Sb, Sb.off_p + I.vb[k]);
          if (both || cross) continue;
          D.mults.push_back({f, k, -1});
        }
      }
    }
    if (pass == 0) D.n_lambda_u = (int)D.mults.size();
  }
  D.n_lambda = (int)D.mults.size();
  // G / Gc per subdomain
  std::map<std::tuple<int, int, int>, int> mid;
  for (int i = 0; i < D.n_lambda; ++i) mid[{D.mults[i].iface, D.mults[i].k, D.mults[i].comp}] = i;
  std::vector<std::vector<Trip>> tg(D.subs.size()), tc(D.subs.size());
  auto put = [&](int sub, int row, int sidx, double v, double sign) {
    const Sub& S = D.subs[sub];
    if (S.cpos[sidx] >= 0)
      tc[sub].push_back({row, S.cpos[sidx], sign * v});
    else
      tg[sub].push_back({row, sidx, sign * v});
  };
  for (int f = 0; f < (int)D.ifs.size(); ++f) {
    const Iface& I = D.ifs[f];
    const Sub &Sa = D.subs[I.a], &Sb = D.subs[I.b];
    for (int j = 0; j + 1 < (int)I.va.size(); ++j) {
      const V2 pa = Sa.mesh.vtx[I.va[j]], pb = Sa.mesh.vtx[I.va[j + 1]];
      const Dense H = local_interface(pa, pb, cfg.order);
      std::vector<int> na = {I.va[j], I.va[j + 1]}, nb = {I.vb[j], I.vb[j + 1]};
      if (cfg.order == 2) na.push_back(Sa.mesh.nv() + I.ea[j]), nb.push_back(Sb.mesh.nv() + I.eb[j]);
      for (int i = 0; i < 2; ++i)
        for (int c = 0; c < 2; ++c) {
          auto it = mid.find({f, j + i, c});
          if (it == mid.end()) continue;
          for (int q = 0; q < (int)na.size(); ++q) {
            put(I.a, it->second, Sa.off_u + Sa.u.dof(na[q], c), H(i, q), +1.0);
            put(I.b, it->second, Sb.off_u + Sb.u.dof(nb[q], c), H(i, q), -1.0);
          }
        }
      if (I.pp) {
        const Dense H1 = local_interface(pa, pb, 1);
        for (int i = 0; i < 2; ++i) {
          auto it = mid.find({f, j + i, -1});
          if (it == mid.end()) continue;
          for (int q = 0; q < 2; ++q) {
            put(I.a, it->second, Sa.off_p + na[q], H1(i, q), +1.0);
            put(I.b, it->second, Sb.off_p + nb[q], H1(i, q), -1.0);
          }
        }
      }
    }
  }
  for (std::size_t s = 0; s < D.subs.size(); ++s) {
    Sub& S = D.subs[s];
    S.G = Csr::from_trips(D.n_lambda, S.dim, tg[s]);
    S.Gc = Csr::from_trips(D.n_lambda, (int)S.cons.size(), tc[s]);
    // Dirichlet-preconditioner boundary sets (feti.hpp:178-200 generalised)
    for (int nd = 0; nd < S.u.nnode; ++nd)
      if (S.u.on_iface[nd])
        for (int c = 0; c < 2; ++c)
          if (S.cpos[S.off_u + S.u.dof(nd, c)] < 0) S.Bu.push_back(S.off_u + S.u.dof(nd, c));
  }
  for (const Iface& I : D.ifs) {
    if (!I.pp) continue;
    for (int side = 0; side < 2; ++side) {
      Sub& S = D.subs[side ? I.b : I.a];
      for (int v : side ? I.vb : I.va)
        if (S.cpos[S.off_p + v] < 0) S.Bp.push_back(S.off_p + v);
    }
  }
  for (auto& S : D.subs) {
    std::sort(S.Bp.begin(), S.Bp.end());
    S.Bp.erase(std::unique(S.Bp.begin(), S.Bp.end()), S.Bp.end());
  }
  return D;
}

/// Loads at time t (assembly.hpp:430-540): body force, traction, source Z,
/// boundary flux.  F has n_u entries, Z has n_s entries (P only).
inline void assemble_loads(const Disc& D, const Sub& S, double t, Vec& F, Vec& Z) {
  const Mesh& m = S.mesh;
  F.assign(S.n_u, 0.0);
  Z.assign(S.n_s, 0.0);
  const Quad q = triangle_rule(kFormDegree);
  const VFn& f = S.region == Region::P ? D.sc.f_P : D.sc.f_E;
  double v[6], sv[3];
  V2 g[6], sg[3];
  for (int tr = 0; tr < m.nt(); ++tr) {
    const auto c = m.coords(tr);
    const Affine A(c);
    const auto nodes = detail::local_u_nodes(m, tr, S.u.order);
    const bool src = !D.src_elem.empty() && D.src_elem[S.gelem[tr]];
    for (int k = 0; k < q.size(); ++k) {
      eval_basis(S.u.order, q.pts[k], v, g);
      const V2 x = A.map(c[0], q.pts[k]);
      const V2 fx = f(x, t);
      const double w = q.w[k] * std::abs(A.det);
      for (std::size_t i = 0; i < nodes.size(); ++i) {
        F[S.u.dof(nodes[i], 0)] += w * v[i] * fx.x;
        F[S.u.dof(nodes[i], 1)] += w * v[i] * fx.y;
      }
      if (S.region == Region::P) {
        eval_basis(1, q.pts[k], sv, sg);
        const double zq = D.sc.per_element ? (src ? D.sc.src_rate : 0.0) : D.sc.z(x, t);
        for (int i = 0; i < 3; ++i) Z[m.tri[tr][i]] += w * sv[i] * zq;
      }
    }
  }
  const Quad e5 = edge_rule(5);
  const VFn& trac = S.region == Region::P ? D.sc.tr_P : D.sc.tr_E;
  for (const auto& be : m.bnd) {
    if (be.tag.interface_edge) continue;
    const V2 a = m.vtx[m.edge[be.edge][0]], b = m.vtx[m.edge[be.edge][1]];
    const double L = (b - a).norm();
    std::vector<int> nodes = {m.edge[be.edge][0], m.edge[be.edge][1]};
    if (S.u.order == 2) nodes.push_back(m.nv() + be.edge);
    for (int k = 0; k < e5.size(); ++k) {
      const double s = e5.pts[k].x;
      double ev[3];
      eval_edge_basis(S.u.order, s, ev);
      const V2 x = a + (b - a) * s;
      const V2 tx = trac(x, t);
      const double w = e5.w[k] * L;
      for (std::size_t i = 0; i < nodes.size(); ++i) {
        F[S.u.dof(nodes[i], 0)] += w * ev[i] * tx.x;
        F[S.u.dof(nodes[i], 1)] += w * ev[i] * tx.y;
      }
    }
    if (S.region == Region::P && be.tag.pressure == PTag::flux) {
      for (int k = 0; k < e5.size(); ++k) {
        const double s = e5.pts[k].x;
        double ev[2];
        eval_edge_basis(1, s, ev);
        const double zw = D.sc.flux(a + (b - a) * s, t);
        const double w = e5.w[k] * L;
        Z[m.edge[be.edge][0]] += w * ev[0] * zw;
        Z[m.edge[be.edge][1]] += w * ev[1] * zw;
      }
    }
  }
}

struct StepRhs {
  std::vector<Vec> b, g;
  Vec d;
};

/// assemble_rhs_step (assembly.hpp:550-579): b_P = [F | 0 | 0 | -R eta_prev - tau Z],
/// b_E = [F | 0], lifting, d = -sum_s Gc_s g_s.
inline StepRhs assemble_rhs(const Disc& D, double t, const std::vector<Vec>& eta_prev) {
  StepRhs r;
  r.b.resize(D.subs.size());
  r.g.resize(D.subs.size());
  r.d.assign(D.n_lambda, 0.0);
  for (std::size_t s = 0; s < D.subs.size(); ++s) {
    const Sub& S = D.subs[s];
    Vec F, Z;
    assemble_loads(D, S, t, F, Z);
    Vec& b = r.b[s];
    b.assign(S.dim, 0.0);
    for (int i = 0; i < S.n_u; ++i) b[S.off_u + i] = F[i];
    if (S.region == Region::P) {
      const Vec Re = S.R.mul(eta_prev[s]);
      for (int i = 0; i < S.n_s; ++i) b[S.off_p + i] = -Re[i] - D.tau * Z[i];
    }
    Vec& g = r.g[s];
    g.resize(S.cons.size());
    for (std::size_t k = 0; k < S.cons.size(); ++k) {
      const Cons& c = S.cons[k];
      if (c.is_u) {
        const V2 u = (S.region == Region::P ? D.sc.u_bc_P : D.sc.u_bc_E)(c.xy, t);
        g[k] = c.comp == 0 ? u.x : u.y;
      } else {
        g[k] = D.sc.p_bc(c.xy, t);
      }
    }
    if (!S.cons.empty()) {
      S.lift.mv(g.data(), b.data(), true, -1.0);
      for (std::size_t k = 0; k < S.cons.size(); ++k) b[S.cons[k].sidx] = g[k];
      S.Gc.mv(g.data(), r.d.data(), true, -1.0);
    }
  }
  return r;
}

}  // namespace oracle
