// TEST INFRASTRUCTURE ONLY — see o_core.hpp.
// oracle_capi.cpp — extern "C" surface of the CPU oracle for the pytest
// checker (ctypes) and bench.py's cpu_baseline leg.  Never linked by the
// product library.
#include <atomic>
#include <cstring>
#include <memory>

#include "o_feti.hpp"
#include "o_verify.hpp"

using namespace oracle;

extern "C" {

struct or_config {
  int mesh_n, SX, SY, order;
  double E, nu, alpha, c0, kperm, mu_f, dt;
  int steps;
  int mu_conv;   // 0 paper, 1 standard
  int scenario;  // 0 mms-t, 1 mms, 2 injection, 3 barry-mercer
  int precond;   // 0 identity, 1 generalized, 2 dirichlet
  int krylov;    // 0 auto, 1 pcg, 2 minres
  double tol;
  int max_iter, warm, threads;
  unsigned long long seed;
  double logk_mean, logk_sd;
};
}

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

Config to_cfg(const or_config* c) {
  Config k;
  static const char* sc[] = {"mms-t", "mms", "injection", "barry-mercer"};
  static const char* pr[] = {"identity", "generalized", "dirichlet", "generalized-mortar", "dirichlet-mortar"};
  static const char* kr[] = {"auto", "pcg", "minres", "sqmr"};
  if (c->scenario < 0 || c->scenario > 3 || c->precond < 0 || c->precond > 4 || c->krylov < 0 || c->krylov > 3)
    throw ConfigError("config enum out of range");
  k.scenario = sc[c->scenario];
  k.mesh_n = c->mesh_n, k.SX = c->SX, k.SY = c->SY, k.order = c->order;
  k.E = c->E, k.nu = c->nu, k.alpha = c->alpha, k.c0 = c->c0, k.kperm = c->kperm, k.mu_f = c->mu_f;
  k.dt = c->dt, k.steps = c->steps;
  k.conv = c->mu_conv == 1 ? MuConv::standard : MuConv::paper;
  k.precond = pr[c->precond];
  k.krylov = kr[c->krylov];
  k.tol = c->tol, k.max_iter = c->max_iter, k.warm = c->warm != 0, k.threads = c->threads;
  k.seed = c->seed, k.logk_mean = c->logk_mean, k.logk_sd = c->logk_sd;
  return k;
}

struct Handle {
  Disc D;
  std::unique_ptr<Feti> op;
  std::vector<State> states;
  std::vector<PcgReport> reps;
  double t_setup = 0, t_factor = 0;
  std::vector<double> t_step;
};

std::array<V2, 3> tri_of(const double* t) { return {V2(t[0], t[1]), V2(t[2], t[3]), V2(t[4], t[5])}; }

void copy_dense(const Dense& d, double* out) { std::memcpy(out, d.a.data(), sizeof(double) * d.a.size()); }

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

// ---------------- element / quadrature KATs ----------------
int or_triangle_rule(int degree, double* pts, double* w, int* n) {
  return guard([&] {
    const Quad q = triangle_rule(degree);
    *n = q.size();
    for (int k = 0; k < q.size(); ++k) pts[2 * k] = q.pts[k].x, pts[2 * k + 1] = q.pts[k].y, w[k] = q.w[k];
  });
}
int or_edge_rule(int degree, double* pts, double* w, int* n) {
  return guard([&] {
    const Quad q = edge_rule(degree);
    *n = q.size();
    for (int k = 0; k < q.size(); ++k) pts[k] = q.pts[k].x, w[k] = q.w[k];
  });
}
int or_eval_basis(int order, double x, double y, double* v, double* g) {
  return guard([&] {
    V2 gg[6];
    eval_basis(order, V2(x, y), v, gg);
    for (int i = 0; i < nbasis(order); ++i) g[2 * i] = gg[i].x, g[2 * i + 1] = gg[i].y;
  });
}
int or_local_elastic(const double* tri, double mu, int order, double* out) {
  return guard([&] { copy_dense(local_elastic(tri_of(tri), mu, order), out); });
}
int or_local_div(const double* tri, int order, double* out) {
  return guard([&] { copy_dense(local_div(tri_of(tri), order), out); });
}
int or_local_mass(const double* tri, double* out) {
  return guard([&] { copy_dense(local_mass(tri_of(tri)), out); });
}
int or_local_diffusion(const double* tri, double k00, double k01, double k11, double muf, double* out) {
  return guard([&] { copy_dense(local_diffusion(tri_of(tri), k00, k01, k11, muf), out); });
}
int or_local_interface(double ax, double ay, double bx, double by, int trace_order, double* out) {
  return guard([&] { copy_dense(local_interface(V2(ax, ay), V2(bx, by), trace_order), out); });
}

// ---------------- mesh KATs ----------------
int or_mesh_build(int region, const double* rect, int nx, int ny, void** out) {
  return guard([&] {
    auto* m = new Mesh(build_subdomain_mesh(region == 0 ? Region::P : Region::E,
                                            Rect{rect[0], rect[1], rect[2], rect[3]}, nx, ny));
    *out = m;
  });
}
void or_mesh_free(void* h) { delete static_cast<Mesh*>(h); }
void or_mesh_counts(void* h, int* nv, int* nt, int* ne) {
  auto* m = static_cast<Mesh*>(h);
  *nv = m->nv(), *nt = m->nt(), *ne = m->ne();
}
void or_mesh_vertices(void* h, double* xy) {
  auto* m = static_cast<Mesh*>(h);
  for (int v = 0; v < m->nv(); ++v) xy[2 * v] = m->vtx[v].x, xy[2 * v + 1] = m->vtx[v].y;
}
void or_mesh_triangles(void* h, int* t, double* area) {
  auto* m = static_cast<Mesh*>(h);
  for (int k = 0; k < m->nt(); ++k) {
    for (int i = 0; i < 3; ++i) t[3 * k + i] = m->tri[k][i];
    area[k] = m->area(k);
  }
}
/// rule: 0 all-Dirichlet (+p Dirichlet) with interface at y=param; 1/2 Barry-Mercer P/E;
/// 3 partial (bottom only, else untaggable); 4 clamp everything (no interface).
int or_mesh_tag(void* h, int rule, double param) {
  return guard([&] {
    auto* m = static_cast<Mesh*>(h);
    TagRule r;
    const Params P = make_params(1e4, 0.2, 1e4, 0.2, 1.0, 0.1, 1.0, 1.0);
    const Scenario bm = barry_mercer(P);
    switch (rule) {
      case 0:
        r = [param](const V2& x) -> std::optional<Tag> {
          if (std::abs(x.y - param) < 1e-9) return Tag::iface();
          return Tag::clamp(PTag::dirichlet);
        };
        break;
      case 1:
      case 2: {
        const Region reg = rule == 1 ? Region::P : Region::E;
        r = [bm, reg](const V2& x) -> std::optional<Tag> {
          if (near(x.y, 0.5)) return Tag::iface();
          return bm.outer_tag(reg, x);
        };
        break;
      }
      case 3:
        r = [](const V2& x) -> std::optional<Tag> {
          if (std::abs(x.y) < 1e-9) return Tag::clamp();
          return std::nullopt;
        };
        break;
      default:
        r = [](const V2&) -> std::optional<Tag> { return Tag::clamp(); };
    }
    *m = tag_boundary_facets(*m, r);
  });
}
int or_mesh_boundary(void* h, int* edge, int* mask, int* ptag, int* iface, double* mid) {
  auto* m = static_cast<Mesh*>(h);
  for (std::size_t k = 0; k < m->bnd.size(); ++k) {
    edge[k] = m->bnd[k].edge;
    mask[k] = (int)m->bnd[k].tag.disp_mask;
    ptag[k] = (int)m->bnd[k].tag.pressure;
    iface[k] = m->bnd[k].tag.interface_edge;
    const V2 c = m->mid(m->bnd[k].edge);
    mid[2 * k] = c.x, mid[2 * k + 1] = c.y;
  }
  return (int)m->bnd.size();
}
int or_dofmap(void* h, int kind, int order, int* nnode, int* ndof, char* on_iface) {
  return guard([&] {
    const DofMap d = make_dof_map(*static_cast<Mesh*>(h), (Field)kind, order);
    *nnode = d.nnode, *ndof = d.ndof;
    if (on_iface) std::memcpy(on_iface, d.on_iface.data(), d.nnode);
  });
}
int or_pair(void* ha, void* hb, int order, int* npairs, int* pairs, int* nmult, int* nedges) {
  return guard([&] {
    const Mesh &a = *static_cast<Mesh*>(ha), &b = *static_cast<Mesh*>(hb);
    const Pairing p = pair_interface(a, b, make_dof_map(a, Field::disp, order), make_dof_map(b, Field::disp, order));
    *npairs = (int)p.node_pairs.size();
    if (pairs)
      for (std::size_t k = 0; k < p.node_pairs.size(); ++k)
        pairs[2 * k] = p.node_pairs[k].first, pairs[2 * k + 1] = p.node_pairs[k].second;
    *nmult = (int)p.mult_vertices_a.size();
    *nedges = p.n_edges;
  });
}

// ---------------- discretisation / FETI ----------------
int or_create(const or_config* c, void** out) {
  return guard([&] {
    auto h = std::make_unique<Handle>();
    const auto t0 = std::chrono::steady_clock::now();
    h->D = build_discretization(to_cfg(c));
    const auto t1 = std::chrono::steady_clock::now();
    h->op = std::make_unique<Feti>(h->D);
    const auto t2 = std::chrono::steady_clock::now();
    h->t_setup = std::chrono::duration<double>(t1 - t0).count();
    h->t_factor = std::chrono::duration<double>(t2 - t1).count();
    h->states.push_back(project_initial(h->D));
    *out = h.release();
  });
}
void or_destroy(void* h) { delete static_cast<Handle*>(h); }

/// info: [n_sub, n_lambda, n_lambda_u, n_coarse, minres, N, n_floating]
void or_info(void* hh, int* info, double* dinfo) {
  auto* h = static_cast<Handle*>(hh);
  int nf = 0;
  for (auto& S : h->D.subs) nf += S.floating;
  info[0] = (int)h->D.subs.size();
  info[1] = h->D.n_lambda;
  info[2] = h->D.n_lambda_u;
  info[3] = h->op->n_coarse();
  info[4] = h->op->krylov_kind();
  info[5] = h->D.N;
  info[6] = nf;
  // dinfo: [tau, T, t_setup, t_factor, lam_P, mu_P, k1, k2, k3]
  dinfo[0] = h->D.tau;
  dinfo[1] = h->D.T;
  dinfo[2] = h->t_setup;
  dinfo[3] = h->t_factor;
  dinfo[4] = h->D.par.lam_P;
  dinfo[5] = h->D.par.mu_P;
  dinfo[6] = h->D.par.k1;
  dinfo[7] = h->D.par.k2;
  dinfo[8] = h->D.par.k3;
}
/// sub info: [region, dim, n_u, n_s, off_u, off_eta, off_xi, off_p, floating, nnzK, n_cons, nnzL(lo32), nBu, nBp]
void or_sub_info(void* hh, int s, long long* info) {
  auto* h = static_cast<Handle*>(hh);
  const Sub& S = h->D.subs[s];
  long long v[] = {S.region == Region::P ? 0 : 1, S.dim, S.n_u, S.n_s, S.off_u, S.off_eta, S.off_xi, S.off_p,
                   S.floating, S.K.nnz(), (long long)S.cons.size(), h->op->factor(s).nnz_L(),
                   (long long)S.Bu.size(), (long long)S.Bp.size()};
  std::memcpy(info, v, sizeof(v));
}
/// which: 0 K, 1 G, 2 Gc, 3 lift, 4 A, 5 B, 6 R, 7 Af.  Call with ptr==nullptr to get nnz/rows/cols.
int or_sub_matrix(void* hh, int s, int which, int* nr, int* nc, int* nnz, int* ptr, int* col, double* val) {
  auto* h = static_cast<Handle*>(hh);
  const Sub& S = h->D.subs[s];
  const Csr* m[] = {&S.K, &S.G, &S.Gc, &S.lift, &S.A, &S.B, &S.R, &S.Af};
  if (which < 0 || which > 7) return 4;
  const Csr& M = *m[which];
  *nr = M.nr, *nc = M.nc, *nnz = M.nnz();
  if (ptr) {
    std::memcpy(ptr, M.ptr.data(), sizeof(int) * (M.nr + 1));
    std::memcpy(col, M.col.data(), sizeof(int) * M.nnz());
    std::memcpy(val, M.val.data(), sizeof(double) * M.nnz());
  }
  return 0;
}
/// multiplier table: (iface, k, comp) per lambda; interface table (a, b, horiz, pp)
void or_mults(void* hh, int* m, int* ifs) {
  auto* h = static_cast<Handle*>(hh);
  for (int i = 0; i < h->D.n_lambda; ++i)
    m[3 * i] = h->D.mults[i].iface, m[3 * i + 1] = h->D.mults[i].k, m[3 * i + 2] = h->D.mults[i].comp;
  if (ifs)
    for (std::size_t f = 0; f < h->D.ifs.size(); ++f)
      ifs[4 * f] = h->D.ifs[f].a, ifs[4 * f + 1] = h->D.ifs[f].b, ifs[4 * f + 2] = h->D.ifs[f].horiz,
                ifs[4 * f + 3] = h->D.ifs[f].pp;
}
int or_n_ifaces(void* hh) { return (int)static_cast<Handle*>(hh)->D.ifs.size(); }
void or_kelem(void* hh, double* k) {
  auto* h = static_cast<Handle*>(hh);
  std::memcpy(k, h->D.kelem.data(), sizeof(double) * h->D.kelem.size());
}
int or_n_src(void* hh) {
  auto* h = static_cast<Handle*>(hh);
  int n = 0;
  for (char c : h->D.src_elem) n += c;
  return n;
}

int or_apply(void* hh, const double* x, double* y) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    const Vec v(x, x + h->D.n_lambda);
    const Vec r = h->op->apply(v);
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int or_precond(void* hh, const double* x, double* y) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    const Vec v(x, x + h->D.n_lambda);
    const Vec r = h->op->precondition(v);
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int or_apply_subset(void* hh, const double* x, double* y, const int* subs, int nsubs, int which) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    const Vec v(x, x + h->D.n_lambda);
    const Vec r = h->op->apply_subset(v, std::vector<int>(subs, subs + nsubs), which);
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}

int or_project(void* hh, double* x) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    Vec v(x, x + h->D.n_lambda);
    h->op->project(v);
    std::memcpy(x, v.data(), sizeof(double) * v.size());
  });
}
int or_local_solve(void* hh, int s, double* x) {
  return guard([&] { static_cast<Handle*>(hh)->op->local_solve(s, x); });
}

/// Step RHS at time t from the state at `step` (b per subdomain concatenated, d, F).
int or_step_rhs(void* hh, int step, double* b_cat, double* d, double* F) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    const State& st = h->states.at(step);
    const StepRhs r = assemble_rhs(h->D, h->D.time(st.step + 1), eta_of(h->D, st));
    std::size_t o = 0;
    for (auto& b : r.b) {
      if (b_cat) std::memcpy(b_cat + o, b.data(), sizeof(double) * b.size());
      o += b.size();
    }
    if (d) std::memcpy(d, r.d.data(), sizeof(double) * r.d.size());
    if (F) {
      const Vec f = h->op->interface_rhs(r);
      std::memcpy(F, f.data(), sizeof(double) * f.size());
    }
  });
}

/// Advance nsteps from the last stored state; stores every state.
int or_run(void* hh, int nsteps) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    for (int k = 0; k < nsteps; ++k) {
      PcgReport rep;
      const auto t0 = std::chrono::steady_clock::now();
      State nx = advance(h->D, *h->op, h->states.back(), rep);
      h->t_step.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      h->states.push_back(std::move(nx));
      h->reps.push_back(rep);
    }
  });
}
int or_n_states(void* hh) { return (int)static_cast<Handle*>(hh)->states.size(); }
int or_state(void* hh, int step, int s, double* x) {
  auto* h = static_cast<Handle*>(hh);
  if (step < 0 || step >= (int)h->states.size()) return 4;
  const Vec& v = h->states[step].x[s];
  std::memcpy(x, v.data(), sizeof(double) * v.size());
  return 0;
}
/// verify.hpp:62-74 on time level `step`: displacement / pressure L2 errors
int or_errors(void* hh, int step, double* eu, double* ep) {
  auto* h = static_cast<Handle*>(hh);
  if (step < 0 || step >= (int)h->states.size()) return 4;
  return guard([&] { snapshot_errors(h->D, h->states[step], *eu, *ep); });
}
int or_lambda(void* hh, int step, double* l) {
  auto* h = static_cast<Handle*>(hh);
  if (step < 0 || step >= (int)h->states.size()) return 4;
  std::memcpy(l, h->states[step].lambda.data(), sizeof(double) * h->states[step].lambda.size());
  return 0;
}
/// true residual ||P(rhs - F lambda)|| / ||r0|| and SQMR restarts of step k>=1
int or_report_true(void* hh, int step, double* true_res, int* restarts) {
  auto* h = static_cast<Handle*>(hh);
  if (step < 1 || step > (int)h->reps.size()) return 4;
  *true_res = h->reps[step - 1].true_residual, *restarts = h->reps[step - 1].restarts;
  return 0;
}
/// report of step k>=1: iterations, converged, rel_residual, wall seconds; history into hist (may be null)
int or_report(void* hh, int step, int* iters, int* conv, double* rel, double* secs, double* hist, int* nhist) {
  auto* h = static_cast<Handle*>(hh);
  if (step < 1 || step > (int)h->reps.size()) return 4;
  const PcgReport& r = h->reps[step - 1];
  *iters = r.iterations, *conv = r.converged, *rel = r.rel_residual, *secs = h->t_step[step - 1];
  *nhist = (int)r.history.size();
  if (hist) std::memcpy(hist, r.history.data(), sizeof(double) * r.history.size());
  return 0;
}

/// Monolithic solve of the first step from the initial state.
int or_monolithic_step(void* hh, double* x_cat, double* lambda) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hh);
    const State& st = h->states.at(0);
    const StepRhs r = assemble_rhs(h->D, h->D.time(1), eta_of(h->D, st));
    std::vector<Vec> x;
    Vec l;
    monolithic_solve(h->D, r, x, l);
    std::size_t o = 0;
    for (auto& v : x) {
      std::memcpy(x_cat + o, v.data(), sizeof(double) * v.size());
      o += v.size();
    }
    std::memcpy(lambda, l.data(), sizeof(double) * l.size());
  });
}

}  // extern "C"
