// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// o_mesh.hpp — restatement of mesh.hpp: structured triangulation
// (mesh.hpp:104-131), edge discovery (:73-87), boundary tagging (:137-152),
// dof maps (:157-199) and two-sided interface pairing (:255-303).
#pragma once

#include <functional>
#include <map>
#include <optional>

#include "o_core.hpp"

namespace oracle {

enum class Region { P, E };

struct Rect {
  double x0 = 0, y0 = 0, x1 = 1, y1 = 1;
  double w() const { return x1 - x0; }
  double h() const { return y1 - y0; }
};

enum class PTag { none, dirichlet, flux };

/// Boundary classification of one edge (mesh.hpp:20-32).
struct Tag {
  unsigned disp_mask = 0;  // bit c: component c essential
  PTag pressure = PTag::none;
  bool interface_edge = false;
  static Tag clamp(PTag p = PTag::none) { return {3u, p, false}; }
  static Tag iface() { return {0u, PTag::none, true}; }
  bool essential(int c) const { return (disp_mask >> c) & 1u; }
};

struct BEdge {
  int edge = -1;
  Tag tag;
};

struct Mesh {
  Region region = Region::P;
  Rect rect;
  int nx = 0, ny = 0;
  std::vector<V2> vtx;
  std::vector<std::array<int, 3>> tri;
  std::vector<std::array<int, 2>> edge;   // (lo, hi)
  std::vector<std::array<int, 3>> tedge;  // edge opposite local vertex i
  std::vector<BEdge> bnd;
  bool tagged = false;

  int nv() const { return (int)vtx.size(); }
  int nt() const { return (int)tri.size(); }
  int ne() const { return (int)edge.size(); }
  double area(int t) const {
    const V2 a = vtx[tri[t][0]], b = vtx[tri[t][1]], c = vtx[tri[t][2]];
    return 0.5 * ((b.x - a.x) * (c.y - a.y) - (c.x - a.x) * (b.y - a.y));
  }
  V2 mid(int e) const { return (vtx[edge[e][0]] + vtx[edge[e][1]]) * 0.5; }
  std::array<V2, 3> coords(int t) const { return {vtx[tri[t][0]], vtx[tri[t][1]], vtx[tri[t][2]]}; }
};

inline Mesh build_subdomain_mesh(Region region, const Rect& r, int nx, int ny) {
  if (nx < 1 || ny < 1) throw MeshError("build_subdomain_mesh: subdivision counts must be >= 1");
  if (r.w() <= 0 || r.h() <= 0) throw MeshError("build_subdomain_mesh: degenerate rectangle");
  Mesh m;
  m.region = region;
  m.rect = r;
  m.nx = nx;
  m.ny = ny;
  const double hx = r.w() / nx, hy = r.h() / ny;
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) m.vtx.emplace_back(r.x0 + i * hx, r.y0 + j * hy);
  auto id = [nx](int i, int j) { return j * (nx + 1) + i; };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      // cell corners a(i,j) b(i+1,j) c(i+1,j+1) d(i,j+1), split along a-c
      m.tri.push_back({id(i, j), id(i + 1, j), id(i + 1, j + 1)});
      m.tri.push_back({id(i, j), id(i + 1, j + 1), id(i, j + 1)});
    }
  std::map<std::pair<int, int>, int> ids;
  m.tedge.resize(m.tri.size());
  for (std::size_t t = 0; t < m.tri.size(); ++t)
    for (int i = 0; i < 3; ++i) {
      int a = m.tri[t][(i + 1) % 3], b = m.tri[t][(i + 2) % 3];
      if (a > b) std::swap(a, b);
      auto it = ids.find({a, b});
      if (it == ids.end()) {
        it = ids.emplace(std::make_pair(a, b), m.ne()).first;
        m.edge.push_back({a, b});
      }
      m.tedge[t][i] = it->second;
    }
  return m;
}

inline std::vector<int> boundary_edges(const Mesh& m) {
  std::vector<int> cnt(m.ne(), 0);
  for (const auto& te : m.tedge)
    for (int e : te) cnt[e]++;
  std::vector<int> out;
  for (int e = 0; e < m.ne(); ++e)
    if (cnt[e] == 1) out.push_back(e);
  return out;
}

using TagRule = std::function<std::optional<Tag>(const V2&)>;

inline Mesh tag_boundary_facets(Mesh m, const TagRule& rule) {
  m.bnd.clear();
  for (int e : boundary_edges(m)) {
    auto t = rule(m.mid(e));
    if (!t)
      throw MeshError("tag_boundary_facets: untaggable boundary edge at (" +
                      std::to_string(m.mid(e).x) + ", " + std::to_string(m.mid(e).y) + ")");
    m.bnd.push_back({e, *t});
  }
  m.tagged = true;
  return m;
}

enum class Field { disp, xi, eta, p, mult };

/// Nodal layout (mesh.hpp:157-199): P2 node = nv + edge; vector fields
/// interleaved dof = 2*node + c.
struct DofMap {
  Field kind = Field::disp;
  int order = 1, ncomp = 1, nnode = 0, ndof = 0;
  std::vector<V2> xy;
  std::vector<char> on_iface;
  int dof(int node, int c = 0) const { return node * ncomp + c; }
};

inline DofMap make_dof_map(const Mesh& m, Field kind, int order) {
  if (order != 1 && order != 2) throw MeshError("make_dof_map: unsupported polynomial order");
  if (kind != Field::disp && order != 1) throw MeshError("make_dof_map: scalar fields are P1");
  DofMap d;
  d.kind = kind;
  d.order = order;
  d.ncomp = (kind == Field::disp || kind == Field::mult) ? 2 : 1;
  d.nnode = m.nv() + (order == 2 ? m.ne() : 0);
  d.ndof = d.nnode * d.ncomp;
  d.xy.resize(d.nnode);
  for (int v = 0; v < m.nv(); ++v) d.xy[v] = m.vtx[v];
  if (order == 2)
    for (int e = 0; e < m.ne(); ++e) d.xy[m.nv() + e] = m.mid(e);
  d.on_iface.assign(d.nnode, 0);
  for (const auto& b : m.bnd) {
    if (!b.tag.interface_edge) continue;
    d.on_iface[m.edge[b.edge][0]] = 1;
    d.on_iface[m.edge[b.edge][1]] = 1;
    if (order == 2) d.on_iface[m.nv() + b.edge] = 1;
  }
  return d;
}

/// Two-subdomain pairing as in mesh.hpp:255-303 (horizontal interface only;
/// kept for the reference's own mesh tests).
struct Pairing {
  std::vector<std::pair<int, int>> node_pairs;
  std::vector<std::array<int, 4>> edges;  // (edge_a, edge_b, ...) unused detail
  std::vector<int> mult_vertices_a;
  int n_edges = 0;
};

inline Pairing pair_interface(const Mesh& ma, const Mesh& mb, const DofMap& ua, const DofMap& ub) {
  auto trace = [](const DofMap& u) {
    std::vector<int> n;
    for (int i = 0; i < u.nnode; ++i)
      if (u.on_iface[i]) n.push_back(i);
    std::stable_sort(n.begin(), n.end(), [&](int a, int b) { return u.xy[a].x < u.xy[b].x; });
    if (n.empty()) throw MeshError("pair_interface: mesh has no interface edges");
    return n;
  };
  const auto na = trace(ua), nb = trace(ub);
  if (na.size() != nb.size())
    throw NonConformingInterfaceError("pair_interface: trace node counts differ");
  Pairing p;
  for (std::size_t i = 0; i < na.size(); ++i) {
    if ((ua.xy[na[i]] - ub.xy[nb[i]]).linf() > kGeomTol)
      throw NonConformingInterfaceError("pair_interface: interface node mismatch");
    p.node_pairs.emplace_back(na[i], nb[i]);
  }
  for (int n : na)
    if (n < ma.nv()) p.mult_vertices_a.push_back(n);
  int ea = 0, eb = 0;
  for (const auto& b : ma.bnd) ea += b.tag.interface_edge;
  for (const auto& b : mb.bnd) eb += b.tag.interface_edge;
  if (ea != eb) throw NonConformingInterfaceError("pair_interface: interface edge counts differ");
  p.n_edges = ea;
  return p;
}

}  // namespace oracle
