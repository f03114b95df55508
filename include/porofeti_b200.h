/* porofeti_b200.h — C ABI of the B200-native FETI engine
 * (paper_2509_06673_b200/_lib/libporofeti_b200.so).
 *
 * Drop-in boundary for the reference's per-time-step FETI path
 * (/root/reference/proj/include/porofeti).  The reference is a header-only
 * C++ library with Eigen types and no FFI; each entry point below replaces the
 * C++ call named beside it.  Plain pointers and sizes only; all device memory
 * is owned by the context; one CUDA stream per context; calls on one context
 * are serialised.  Every entry point returns a status code:
 *   PF_OK 0, PF_SINGULAR 1 (SingularSubproblemError, core.hpp:52),
 *   PF_BREAKDOWN 2 (PcgBreakdownError, core.hpp:57),
 *   PF_NOT_CONVERGED 3 (SolverError, core.hpp:62),
 *   PF_INVALID 4 (MeshError/AssemblyError/ConfigError, core.hpp:37-70),
 *   PF_CUDA 5 (no device / CUDA failure — there is no CPU fallback),
 *   PF_INTERNAL 99.
 * Vectors in the "saddle" layout follow the reference's per-subdomain saddle
 * order: P = [u, eta, xi, p], E = [u, xi] (assembly.hpp:338-398); u is
 * interleaved node-major (mesh.hpp:157-199).
 */
#ifndef POROFETI_B200_H
#define POROFETI_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_SINGULAR 1
#define PF_BREAKDOWN 2
#define PF_NOT_CONVERGED 3
#define PF_INVALID 4
#define PF_CUDA 5
#define PF_INTERNAL 99

/* scenario ids */
#define PF_SCEN_MMS_T 0        /* BASELINE configs 1-4: time-linear MMS */
#define PF_SCEN_MMS 1          /* reference stationary MMS (model.hpp:146) */
#define PF_SCEN_INJECTION 2    /* BASELINE config 5 */
#define PF_SCEN_BARRY_MERCER 3 /* reference Barry-Mercer (model.hpp:274) */
/* preconditioners: identity, generalized (feti.hpp:86-88,131), dirichlet
 * (feti-schur, feti.hpp:133-141), and the mortar-scaled variants */
#define PF_PREC_IDENTITY 0
#define PF_PREC_GENERALIZED 1
#define PF_PREC_DIRICHLET 2
#define PF_PREC_GENERALIZED_MORTAR 3
#define PF_PREC_DIRICHLET_MORTAR 4
/* Krylov: auto = reference PCG (feti.hpp:263) when no pressure multipliers,
 * SQMR otherwise */
#define PF_KRYLOV_AUTO 0
#define PF_KRYLOV_PCG 1
#define PF_KRYLOV_MINRES 2
#define PF_KRYLOV_SQMR 3
/* direct interface solve, the GPU analogue of the reference's monolithic
 * solver (SolverChoice::monolithic, feti.hpp:313-440, timeloop.hpp:139-160):
 * the coupled system condensed exactly onto the multipliers — no Krylov
 * iterations; the same fields as the reference's direct solve.  Up to 4096
 * multipliers the interface operator is inverted densely (one GEMV per step);
 * beyond, it is factorised sparsely: a multifrontal block LDL^T over a nested
 * dissection of the subdomain grid, whose fronts are condensed on the FP64
 * tensor cores and applied as one HBM-bound GEMV launch per tree depth
 * (BASELINE c4: 162,378 multipliers, 1023 fronts).  PF_DIRECT=dense|sparse in
 * the environment overrides the size rule (tests). */
#define PF_KRYLOV_DIRECT 4

/* Run configuration (reference RunConfig, config.hpp:17-43, plus the
 * partition).  Same field order as the oracle's or_config. */
typedef struct pf_config {
  int mesh_n, SX, SY, order;
  double E, nu, alpha, c0, kperm, mu_f, dt;
  int steps;
  int mu_conv;  /* 0 paper mu=E/(1+nu) (model.hpp:30), 1 standard */
  int scenario;
  int precond;
  int krylov;
  double tol;
  int max_iter, warm, threads;
  unsigned long long seed;
  double logk_mean, logk_sd;
} pf_config;

typedef struct pf_info {
  int n_sub, n_lambda, n_lambda_u, n_coarse, krylov, N, n_floating, n_types;
  long long total_dim, nnz_L, nnz_L_interior, nnz_K, n_supernodes, n_tasks;
  double tau, T;
  double t_setup, t_assemble, t_factor, t_upload;
  double bytes_fapply;  /* algorithmic bytes of one F-apply (SURVEY §8d B_F) */
  double bytes_precond; /* algorithmic bytes of one preconditioner apply */
  int n_levels;         /* task levels of the subdomain sweep schedule */
  int dual;             /* 1: explicit local dual operators (F-apply / Dirichlet as dense GEMVs) */
  double bytes_symv;    /* algorithmic bytes of one k_local_symv launch (n(n+1)/2 values per operator) */
  double bytes_symv_stored; /* bytes it streams (packed 32x32 tiles incl. padding) */
  double bytes_qsolve;  /* operator bytes of one mortar Gram solve (dense units + dense top), as stored
                           (bitwise-equal unit operators kept once) */
  double bytes_qsolve_applied; /* operator bytes one solve applies (every unit counted) */
  double bytes_flocal;  /* bytes of one local dual-operator product (type-shared copies once + per-subdomain
                           operators + gathered inputs, their indices and the local results) */
  double flops_flocal;  /* its flops (2 n^2 per subdomain) */
  double bytes_coarse;  /* bytes of one dense coarse GEMV ((G_c^T G_c)^-1, n_c^2 values) */
  double bytes_factor_stored; /* factor values stored for the per-step sweeps (after same-type sharing) */
  double flops_backsub;  /* explicit back-substitution GEMM per step (0: the sweep back-substitutes) */
  double bytes_backsub;  /* its operator + vector bytes */
  double bytes_direct;   /* krylov = direct: operator bytes one interface solve reads (dense [Z | Y_c], or the
                            front operators M, T of the sparse variant plus Y_c), each once */
  double t_direct_setup; /* its setup (factorisation / inversion) in seconds */
  int direct_sparse;     /* 1: multifrontal factorisation over the subdomain grid (pf_iface.hpp) */
  int direct_fronts;     /* its fronts */
  int sweep_width;       /* same-type subdomains per warp task of the per-step factor sweep (1: scalar sweep;
                            2 / 4: wide sweep, each factor value applied to that many right-hand sides) */
  int sweep_wide_problems; /* groups of sweep_width subdomains (padded) the wide sweep runs */
  int q_local;           /* 1: the mortar Gram solve runs edge-local (explicit (interface, component) block
                            inverses + cross-point corrections, two launches); 0: generic sparse factor */
  int q_local_blocks;    /* its blocks */
  double q_local_drop;   /* the relative far-corner coupling of the block inverses it drops (checked <= 1e-9) */
} pf_info;

typedef struct pf_sub_info {
  int region, dim, n_u, n_s, off_u, off_eta, off_xi, off_p, floating, n_cons, type;
  long long nnz_L;
} pf_sub_info;

/* PcgReport (feti.hpp:59-67) + device timings */
typedef struct pf_report {
  int step, iterations, converged, method; /* method: 1 pcg, 2 minres, 3 sqmr, 4 direct */
  double rel_residual;
  double seconds;     /* device time of the whole advance (CUDA events) */
  double t_rhs, t_krylov, t_back;
  int f_applies, precond_applies;
  /* ||P(rhs - F lambda)|| / ||P rhs|| of the returned multiplier, recomputed
   * with one extra F-apply.  SQMR: part of the convergence test — the
   * quasi-residual (rel_residual, relative to the warm-started residual like
   * REF's criterion) only estimates the residual, so a step converges when
   * that estimate is below tol AND this true residual is below tol.  PCG:
   * reported beside REF's sqrt(r.z). */
  double true_residual;
  int restarts; /* SQMR: true-residual checks that failed (iteration continued with a tighter estimate threshold) */
} pf_report;

typedef struct pf_ctx pf_ctx;

/* build_discretization (timeloop.hpp:51) + StepSolver ctor (timeloop.hpp:137)
 * + FetiOperator ctor (feti.hpp:76): partition, device assembly, per-subdomain
 * factorisation with the seeded residual check (feti.hpp:28-36), projection of
 * the initial state (timeloop.hpp:75). */
int pf_create(pf_ctx** out, const pf_config* cfg);
/* Same, with an explicit per-element permeability array (2*n*n values, global
 * element order) overriding the seeded generator of the injection scenario. */
int pf_create_with_permeability(pf_ctx** out, const pf_config* cfg, const double* k_elem);

/* Multi-GPU sharding: one process per GPU, rank r owns the
 * subdomains s with s % nranks == r; every lambda-space partial result
 * (F-apply, preconditioner, interface right-hand side, rigid right-hand side)
 * is summed over ranks with ncclAllReduce on the context stream (nccl_id: the
 * 128-byte ncclUniqueId from pf_nccl_unique_id on rank 0, broadcast by the
 * host), or with a host-provided reducer (pf_set_reducer: called with a HOST
 * copy of the partial vector, which it must overwrite with the sum over
 * ranks, e.g. via MPI or gloo).  Krylov vectors are replicated; reductions are
 * deterministic for a fixed rank count. */
typedef void (*pf_reduce_fn)(void* user, double* host_buf, int n, void* cuda_stream);
int pf_create_sharded(pf_ctx** out, const pf_config* cfg, const double* k_elem, int rank, int nranks,
                      const void* nccl_id);
int pf_nccl_unique_id(void* out128);
int pf_set_reducer(pf_ctx* ctx, pf_reduce_fn fn, void* user);
/* owned subdomains (global ids) into out (may be NULL); returns the count */
int pf_owned_subdomains(const pf_ctx* ctx, int* out);
/* the shard plan itself (host only): owned subdomain ids of `rank`; returns the count */
int pf_shard_plan(int n_sub, int rank, int nranks, int* owned);
void pf_destroy(pf_ctx* ctx);
const char* pf_last_error(const pf_ctx* ctx); /* ctx may be NULL (creation errors) */

int pf_get_info(const pf_ctx* ctx, pf_info* out);
int pf_get_sub_info(const pf_ctx* ctx, int s, pf_sub_info* out);

/* FetiOperator::apply (feti.hpp:101): y = sum_s G_s K_s^+ G_s^T x, host buffers. */
int pf_apply(pf_ctx* ctx, const double* x, double* y);
/* FetiOperator::apply_preconditioner (feti.hpp:127). */
int pf_apply_precond(pf_ctx* ctx, const double* r, double* z);
/* natural coarse projector P = I - G_c (G_c^T G_c)^{-1} G_c^T (in place). */
int pf_project(pf_ctx* ctx, double* x);
/* SubdomainFactorization::solve (feti.hpp:38) of subdomain s, saddle layout, in place. */
int pf_local_solve(pf_ctx* ctx, int s, double* x);
/* FetiOperator::interface_rhs (feti.hpp:147) of the next step from the current state. */
int pf_interface_rhs(pf_ctx* ctx, double* F);

/* StepSolver::advance (timeloop.hpp:150) on the device-resident state. */
int pf_step(pf_ctx* ctx, pf_report* rep);
/* advance with host buffers (the reference signature): prev state in (all
 * subdomains' saddle vectors concatenated + lambda), next state out.  Of
 * prev_x only the eta blocks of the poroelastic subdomains are read (the step's
 * right-hand side needs eta^{n-1}, assembly.hpp:558) plus prev_lambda (warm
 * start, timeloop.hpp:168-169); every other entry may hold anything.  On an
 * error the device-resident state is undefined (neither snapshot) until the
 * next successful pf_set_state / pf_advance. */
int pf_advance(pf_ctx* ctx, const double* prev_x, const double* prev_lambda, int prev_step,
               double* next_x, double* next_lambda, pf_report* rep);
/* state accessors (saddle layout per subdomain; lambda) */
int pf_get_state(pf_ctx* ctx, int s, double* x);
int pf_get_state_all(pf_ctx* ctx, double* x_cat);
int pf_get_lambda(pf_ctx* ctx, double* lambda);
int pf_set_state(pf_ctx* ctx, const double* x_cat, const double* lambda, int step);
int pf_current_step(const pf_ctx* ctx);
/* bytes pf_advance copied host -> device in its last call (the eta blocks and lambda) */
long long pf_last_h2d_bytes(const pf_ctx* ctx);

/* Spatial L2 errors of the current state against the scenario's exact
 * solution — verify.hpp:62-74 (snapshot_u_error: u over every subdomain;
 * snapshot_p_error: the Darcy pressure over the poroelastic ones), computed on
 * the device (degree-4 Dunavant rule, verify.hpp:15, deterministic reduction).
 * The L-inf(L2) error of verify.hpp:77-83 is the maximum over the steps.
 * PF_INVALID for scenarios without an exact solution (injection, Barry-Mercer). */
int pf_errors(pf_ctx* ctx, double* err_u, double* err_p);

/* min / max of the nodal Darcy pressure of the current state over the
 * poroelastic subdomains (the per-snapshot inputs of oscillation_check,
 * verify.hpp:169-195; 0, 0 without a poroelastic subdomain). */
int pf_pressure_range(pf_ctx* ctx, double* pmin, double* pmax);

/* Page-locked host buffers for the host-buffer entry points (pf_advance,
 * pf_set_state, pf_get_state_all): copies from them run at full PCIe/C2C rate. */
int pf_host_alloc(size_t bytes, void** out);
void pf_host_free(void* p);

/* Device-resident micro-benchmarks (CUDA events on the context stream).
 * kind: 0 F-apply, 1 preconditioner, 2 one batched factor sweep (forward +
 * backward over every subdomain), 3 the local dual-operator products alone,
 * 4 one mortar Gram solve Q, 5 one dense coarse GEMV, 6 the operator of the
 * direct interface solve applied once (PF_KRYLOV_DIRECT contexts: the dense
 * [Z | Y_c] GEMV, or F^{-1} through the fronts of the sparse variant), 7 the
 * sparse variant's whole interface solve (fronts + rigid-mode border Y_c). */
int pf_bench_op(pf_ctx* ctx, int kind, int warmup, int iters, double* ms_per_op);
/* tests: wide vs scalar per-step sweep on the current right-hand side; out = (differing entries, max |diff|)
   per elimination-tree level; returns the level count (negative: status) */
int pf_debug_wide_check(pf_ctx* ctx, double* out, int cap);
/* nsteps device-resident StepSolver::advance calls bracketed by CUDA events. */
int pf_bench_steps(pf_ctx* ctx, int nsteps, double* ms_total, int* iters_total, int* fapplies_total);
/* number of kernels this library has launched (process-wide counter). */
long long pf_launch_count(void);
/* dominant-kernel timing of the last pf_bench_op / pf_step: average ms of the
 * factor-sweep kernels per F-apply and the number of launches per F-apply */
int pf_kernel_stats(pf_ctx* ctx, double* sweep_ms, int* launches_per_apply);

/* Setup phase wall times of pf_create (each phase ends with a stream sync):
 * names joined by ';' into names (cap bytes, may be NULL), seconds into secs
 * (may be NULL; room for the returned count, <= 32). */
int pf_setup_phases(const pf_ctx* ctx, char* names, int cap, double* secs);

/* Per-kernel timing of the sweeps (see pf_engine.cu): 10 doubles. */
int pf_phase_stats(pf_ctx* ctx, int iters, double* out);

/* Element-level entry point (elements.hpp:152-230) evaluated on the device by
 * the same device functions the assembly kernel uses: tri = 3 vertices
 * (x0,y0,x1,y1,x2,y2); outputs row-major: local_elastic_matrix 2nb x 2nb,
 * local_div_matrix 3 x 2nb, local_mass_matrix 3 x 3, local_diffusion_matrix
 * 3 x 3 (K = kperm I); nb = 3 (P1) or 6 (P2).  PF_INVALID for a degenerate
 * triangle (AssemblyError, elements.hpp:139), PF_CUDA without a device. */
int pf_local_matrices(const double* tri, double mu, double kperm, double mu_f, int order,
                      double* elastic, double* div, double* mass, double* diffusion);

/* ---- the reference's per-step pieces, callable one by one -------------------
 * REF StepSolver::advance (timeloop.hpp:150-186) is
 *   rhs = assemble_rhs_step(...)            -> pf_set_loads (optional) + pf_interface_rhs
 *   F = interface_rhs(rhs)                  -> pf_interface_rhs
 *   [lambda, rep] = feti_pcg(op, F, l0, ..) -> pf_krylov
 *   back_substitute(lambda, rhs)            -> pf_back_substitute
 * pf_step / pf_advance run the same sequence on the device in one call. */

/* feti_pcg (feti.hpp:263-308) on a caller right-hand side: the engine's Krylov
 * method (REF PCG without pressure multipliers, SQMR with them; projected onto
 * the natural coarse space when floating subdomains exist, so lambda0 should
 * satisfy G_c^T lambda0 = e) from lambda0 to relative tolerance tol, at most
 * max_iter iterations; lambda_out may alias lambda0.  PF_NOT_CONVERGED when
 * max_iter is reached (lambda_out holds the last iterate, rep is filled),
 * PF_BREAKDOWN on a breakdown (PcgBreakdownError), PF_NOT_CONVERGED also for
 * tol <= 0 (SolverError, feti.hpp:265). */
int pf_krylov(pf_ctx* ctx, const double* rhs, const double* lambda0, double tol, int max_iter,
              double* lambda_out, pf_report* rep);
/* PcgReport::residual_history (feti.hpp:65) of the last solve (pf_krylov or a
 * step): absolute sqrt(r.z) per iteration for PCG, the quasi-residual for
 * SQMR, entry 0 the initial one.  Copies min(count, cap) values into out (may
 * be NULL) and returns the count (negative status on error). */
int pf_last_history(const pf_ctx* ctx, double* out, int cap);

/* FetiOperator::back_substitute (feti.hpp:158-168) for the right-hand side of
 * the last pf_interface_rhs / step: x_s = K_s^+ (b_s - G_s^T lambda) (+ the
 * rigid modes of floating subdomains) for every owned subdomain, saddle layout,
 * concatenated in x_out (total_dim values).  The device state is unchanged. */
int pf_back_substitute(pf_ctx* ctx, const double* lambda, double* x_out);

/* FetiOperator::set_precond (feti.hpp:97): any PF_PREC_* kind; identity always,
 * generalized and the mortar scaling are built on first use, the Dirichlet
 * kinds need the context created with a Dirichlet preconditioner. */
int pf_set_precond(pf_ctx* ctx, int kind);

/* Field-named snapshot (StateSnapshot, state.hpp:8-12; unpack_state,
 * feti.hpp:443-454): field of subdomain s (global id), or of every owned
 * subdomain concatenated in subdomain order with s = -1 (eta and p exist on
 * poroelastic subdomains only).  pf_field_size returns the value count. */
#define PF_FIELD_U 0
#define PF_FIELD_ETA 1
#define PF_FIELD_XI 2
#define PF_FIELD_P 3
int pf_field_size(const pf_ctx* ctx, int field, int s);
int pf_get_field(pf_ctx* ctx, int field, int s, double* out);

/* Caller-supplied loads (StepLoads, assembly.hpp:475-479, + the essential
 * values of assemble_rhs_step, :562-571) in place of the scenario's closed
 * forms.  Layout, owned subdomains in order: F_u n_u values each (body +
 * traction loads on the displacement dofs), Z n_s values per poroelastic
 * subdomain (the mass-balance source row), g the constraint values in
 * pf_get_constraints order (sizes: pf_load_sizes).  NULL = zero.  Applied to
 * the next right-hand side (every later one with persistent != 0, until
 * pf_clear_loads).  pf_scenario_loads returns the scenario's own loads at t in
 * the same layout. */
int pf_get_constraints(const pf_ctx* ctx, int s, int* saddle_index, int* component, double* xy);
int pf_load_sizes(const pf_ctx* ctx, long long* n_F, long long* n_Z, long long* n_g);
int pf_scenario_loads(pf_ctx* ctx, double t, double* F_u, double* Z, double* g);
int pf_set_loads(pf_ctx* ctx, const double* F_u, const double* Z, const double* g, int persistent);
int pf_clear_loads(pf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
