"""B200-native FETI engine for the coupled poroelasticity-elasticity scheme of
arXiv 2509.06673 (reference: /root/reference/proj, header-only C++ `porofeti`).

The product is the shared library ``_lib/libporofeti_b200.so`` (C ABI in
``include/porofeti_b200.h``: CUDA kernels for sm_100a plus the host setup in
C++).  This module is the thin Python host mirror of the reference's
operator interface used by the tests and the benchmark:

    reference (feti.hpp / timeloop.hpp)      here
    ----------------------------------      -----------------------------
    FetiOperator(bs, dofs, variant)          FetiOperator(config)
    FetiOperator::apply                      FetiOperator.apply
    FetiOperator::apply_preconditioner       FetiOperator.apply_preconditioner
    FetiOperator::interface_rhs              FetiOperator.interface_rhs
    StepSolver::advance                      StepSolver.advance
    run_simulation                           run_simulation
    SingularSubproblemError etc.             exceptions below (same names)

There is no CPU fallback: without the compiled library or a CUDA device every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

__all__ = [
    "Config", "make_config", "BASELINE_CONFIGS", "FetiOperator", "StepSolver", "run_simulation",
    "Error", "SingularSubproblemError", "PcgBreakdownError", "SolverError", "ConfigError",
    "CudaUnavailableError", "lib", "build", "LIB_PATH", "oscillation_check", "estimate_order", "mms_errors",
    "convergence_study", "write_error_csv", "write_solver_log_csv", "write_solution_vtk", "barry_mercer_check", "pinned_empty",
    "feti_pcg", "unpack_state", "local_matrices",
]

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# PF_LIB=prof selects the cycle-accounting build (make prof); default: product build
LIB_PATH = os.path.join(PKG, "_lib", "libporofeti_b200" + ("_" + os.environ["PF_LIB"] if os.environ.get("PF_LIB") else "") + ".so")

SCENARIOS = {"mms-t": 0, "mms": 1, "injection": 2, "barry-mercer": 3}
PRECONDS = {"identity": 0, "generalized": 1, "dirichlet": 2, "generalized-mortar": 3, "dirichlet-mortar": 4}
KRYLOV = {"auto": 0, "pcg": 1, "minres": 2, "sqmr": 3, "direct": 4, "monolithic": 4}
METHODS = {1: "pcg", 2: "minres", 3: "sqmr", 4: "direct"}


class Error(RuntimeError):
    code = 99


class SingularSubproblemError(Error):
    code = 1


class PcgBreakdownError(Error):
    code = 2


class SolverError(Error):
    code = 3


class ConfigError(Error):
    code = 4


class CudaUnavailableError(Error):
    code = 5


_ERRORS = {1: SingularSubproblemError, 2: PcgBreakdownError, 3: SolverError, 4: ConfigError,
           5: CudaUnavailableError}


class Config(C.Structure):
    """pf_config (include/porofeti_b200.h)."""

    _fields_ = [
        ("mesh_n", C.c_int), ("SX", C.c_int), ("SY", C.c_int), ("order", C.c_int),
        ("E", C.c_double), ("nu", C.c_double), ("alpha", C.c_double), ("c0", C.c_double),
        ("kperm", C.c_double), ("mu_f", C.c_double), ("dt", C.c_double),
        ("steps", C.c_int), ("mu_conv", C.c_int), ("scenario", C.c_int),
        ("precond", C.c_int), ("krylov", C.c_int),
        ("tol", C.c_double), ("max_iter", C.c_int), ("warm", C.c_int), ("threads", C.c_int),
        ("seed", C.c_ulonglong), ("logk_mean", C.c_double), ("logk_sd", C.c_double),
    ]


class Info(C.Structure):
    _fields_ = [
        ("n_sub", C.c_int), ("n_lambda", C.c_int), ("n_lambda_u", C.c_int), ("n_coarse", C.c_int),
        ("krylov", C.c_int), ("N", C.c_int), ("n_floating", C.c_int), ("n_types", C.c_int),
        ("total_dim", C.c_longlong), ("nnz_L", C.c_longlong), ("nnz_L_interior", C.c_longlong),
        ("nnz_K", C.c_longlong), ("n_supernodes", C.c_longlong), ("n_tasks", C.c_longlong),
        ("tau", C.c_double), ("T", C.c_double),
        ("t_setup", C.c_double), ("t_assemble", C.c_double), ("t_factor", C.c_double), ("t_upload", C.c_double),
        ("bytes_fapply", C.c_double), ("bytes_precond", C.c_double), ("n_levels", C.c_int), ("dual", C.c_int),
        ("bytes_symv", C.c_double), ("bytes_symv_stored", C.c_double), ("bytes_qsolve", C.c_double),
        ("bytes_qsolve_applied", C.c_double), ("bytes_flocal", C.c_double), ("flops_flocal", C.c_double),
        ("bytes_coarse", C.c_double), ("bytes_factor_stored", C.c_double),
        ("flops_backsub", C.c_double), ("bytes_backsub", C.c_double),
        ("bytes_direct", C.c_double), ("t_direct_setup", C.c_double),
        ("direct_sparse", C.c_int), ("direct_fronts", C.c_int),
        ("sweep_width", C.c_int), ("sweep_wide_problems", C.c_int),
        ("q_local", C.c_int), ("q_local_blocks", C.c_int), ("q_local_drop", C.c_double),
    ]


class SubInfo(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("region", "dim", "n_u", "n_s", "off_u", "off_eta", "off_xi",
                                        "off_p", "floating", "n_cons", "type")] + [("nnz_L", C.c_longlong)]


class Report(C.Structure):
    """PcgReport (feti.hpp:59-67) + device timings."""

    _fields_ = [
        ("step", C.c_int), ("iterations", C.c_int), ("converged", C.c_int), ("method", C.c_int),
        ("rel_residual", C.c_double), ("seconds", C.c_double),
        ("t_rhs", C.c_double), ("t_krylov", C.c_double), ("t_back", C.c_double),
        ("f_applies", C.c_int), ("precond_applies", C.c_int),
        ("true_residual", C.c_double), ("restarts", C.c_int),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["method"] = METHODS.get(self.method, str(self.method))
        return d


# BASELINE.json configs; c1 uses the reference's own Dirichlet (feti-schur)
# preconditioner and PCG, c2-c5 the mortar-scaled Dirichlet + SQMR.
# c3 (nu = 0.49999) and c5 (permeability over 6 decades) need ~750 / ~1100
# iterations with this preconditioner, above the reference's default cap of 500.
BASELINE_CONFIGS = {
    "c1": dict(mesh_n=32, SX=1, SY=2, order=1, nu=0.3, c0=1e-3, dt=1e-2, steps=5, scenario="mms-t",
               precond="dirichlet"),
    "c2": dict(mesh_n=128, SX=2, SY=2, order=2, nu=0.3, c0=1e-3, dt=1e-2, steps=10, scenario="mms-t",
               precond="dirichlet-mortar"),
    "c3": dict(mesh_n=512, SX=8, SY=8, order=2, nu=0.49999, c0=1e-3, dt=1e-3, steps=20, scenario="mms-t",
               precond="dirichlet-mortar", max_iter=3000),
    "c4": dict(mesh_n=1024, SX=32, SY=32, order=2, nu=0.3, c0=1e-3, dt=1e-2, steps=10, scenario="mms-t",
               precond="dirichlet-mortar"),
    "c5": dict(mesh_n=512, SX=16, SY=16, order=2, nu=0.4, c0=1e-4, dt=1e-3, steps=100, scenario="injection",
               precond="dirichlet-mortar", max_iter=3000),
}


def make_config(mesh_n=32, SX=1, SY=2, order=1, E=1.0, nu=0.3, alpha=1.0, c0=1e-3, kperm=1.0, mu_f=1.0,
                dt=1e-2, steps=5, mu_conv="paper", scenario="mms-t", precond="dirichlet", krylov="auto",
                tol=1e-10, max_iter=500, warm=True, threads=0, seed=20240901, logk_mean=-2.0, logk_sd=1.0,
                solver=None):
    """`solver`: the reference's SolverChoice name (timeloop.hpp:113-121) --
    "feti-generalized" / "feti-schur" pick the FETI preconditioner (mortar
    scaled on partitions of more than two subdomains), "monolithic" the direct
    interface solve (krylov="direct", the device analogue of MonolithicSolver)."""
    if solver is not None:
        multi = SX * SY > 2
        if solver == "monolithic":
            krylov = "direct"
        elif solver in ("feti-schur", "feti-generalized"):
            base = "dirichlet" if solver == "feti-schur" else "generalized"
            precond, krylov = (base + "-mortar" if multi else base), "auto"
        else:
            raise ConfigError(f"unknown solver {solver!r} (feti-generalized, feti-schur, monolithic)")
    return Config(mesh_n, SX, SY, order, E, nu, alpha, c0, kperm, mu_f, dt, steps,
                  0 if mu_conv == "paper" else 1, SCENARIOS[scenario], PRECONDS[precond], KRYLOV[krylov],
                  tol, max_iter, int(warm), threads, seed, logk_mean, logk_sd)


def build(force=False):
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", PKG], check=True)
    return LIB_PATH


_lib = None


def lib():
    """Load the product library; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaUnavailableError(f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.POINTER(C.c_double)
        L.pf_create.argtypes = [C.POINTER(vp), C.POINTER(Config)]
        L.pf_create_with_permeability.argtypes = [C.POINTER(vp), C.POINTER(Config), vp]
        L.pf_destroy.argtypes = [vp]
        L.pf_last_error.argtypes = [vp]
        L.pf_last_error.restype = C.c_char_p
        L.pf_get_info.argtypes = [vp, C.POINTER(Info)]
        L.pf_get_sub_info.argtypes = [vp, C.c_int, C.POINTER(SubInfo)]
        for name in ("pf_apply", "pf_apply_precond"):
            getattr(L, name).argtypes = [vp, vp, vp]
        L.pf_project.argtypes = [vp, vp]
        L.pf_local_solve.argtypes = [vp, C.c_int, vp]
        L.pf_interface_rhs.argtypes = [vp, vp]
        L.pf_step.argtypes = [vp, C.POINTER(Report)]
        L.pf_advance.argtypes = [vp, vp, vp, C.c_int, vp, vp, C.POINTER(Report)]
        L.pf_get_state.argtypes = [vp, C.c_int, vp]
        L.pf_get_state_all.argtypes = [vp, vp]
        L.pf_get_lambda.argtypes = [vp, vp]
        L.pf_set_state.argtypes = [vp, vp, vp, C.c_int]
        L.pf_current_step.argtypes = [vp]
        L.pf_last_h2d_bytes.argtypes = [vp]
        L.pf_last_h2d_bytes.restype = C.c_longlong
        L.pf_errors.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.pf_pressure_range.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.pf_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
        L.pf_host_free.argtypes = [vp]
        L.pf_bench_op.argtypes = [vp, C.c_int, C.c_int, C.c_int, dp]
        L.pf_debug_wide_check.argtypes = [vp, vp, C.c_int]
        L.pf_kernel_stats.argtypes = [vp, dp, C.POINTER(C.c_int)]
        L.pf_phase_stats.argtypes = [vp, C.c_int, vp]
        L.pf_bench_steps.argtypes = [vp, C.c_int, vp, vp, vp]
        L.pf_launch_count.restype = C.c_longlong
        L.pf_create_sharded.argtypes = [C.POINTER(vp), C.POINTER(Config), vp, C.c_int, C.c_int, vp]
        L.pf_nccl_unique_id.argtypes = [vp]
        L.pf_set_reducer.argtypes = [vp, vp, vp]
        L.pf_owned_subdomains.argtypes = [vp, vp]
        L.pf_shard_plan.argtypes = [C.c_int, C.c_int, C.c_int, vp]
        L.pf_debug_factor_solve.argtypes = [C.c_int, vp, vp, vp, vp, vp, C.c_int, C.c_longlong, vp]
        L.pf_debug_disc.argtypes = [C.POINTER(Config), vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_local_matrices.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_int, vp, vp, vp, vp]
        L.pf_krylov.argtypes = [vp, vp, vp, C.c_double, C.c_int, vp, C.POINTER(Report)]
        L.pf_last_history.argtypes = [vp, vp, C.c_int]
        L.pf_back_substitute.argtypes = [vp, vp, vp]
        L.pf_set_precond.argtypes = [vp, C.c_int]
        L.pf_field_size.argtypes = [vp, C.c_int, C.c_int]
        L.pf_get_field.argtypes = [vp, C.c_int, C.c_int, vp]
        L.pf_get_constraints.argtypes = [vp, C.c_int, vp, vp, vp]
        L.pf_load_sizes.argtypes = [vp, vp, vp, vp]
        L.pf_scenario_loads.argtypes = [vp, C.c_double, vp, vp, vp]
        L.pf_set_loads.argtypes = [vp, vp, vp, vp, C.c_int]
        L.pf_clear_loads.argtypes = [vp]
        L.pf_setup_phases.argtypes = [vp, C.c_char_p, C.c_int, vp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _vec(a, n, what, copy=False):
    """Contiguous float64 copy/view of `a`, checked to hold exactly n values
    (every ABI call reads or writes exactly that many)."""
    a = np.array(a, np.float64) if copy else np.ascontiguousarray(a, np.float64)
    if a.ndim != 1 or a.size != n:
        raise ConfigError(f"{what}: expected a vector of {n} values, got shape {a.shape}")
    return a


def _check(code, ctx=None):
    if code != 0:
        msg = lib().pf_last_error(ctx).decode(errors="replace")
        raise _ERRORS.get(code, Error)(f"[{code}] {msg}")


class FetiOperator:
    """Device-resident FETI interface operator of one discretisation
    (reference FetiOperator, feti.hpp:74-232, plus build_discretization)."""

    def __init__(self, config=None, permeability=None, rank=0, nranks=1, nccl_id=None, **kw):
        self.cfg = config if isinstance(config, Config) else make_config(**kw)
        L = lib()
        h = C.c_void_p()
        if nranks > 1:
            k = None if permeability is None else np.ascontiguousarray(permeability, np.float64)
            idb = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
            code = L.pf_create_sharded(C.byref(h), C.byref(self.cfg), None if k is None else _ptr(k), rank, nranks,
                                       idb)
        elif permeability is not None:
            k = np.ascontiguousarray(permeability, np.float64)
            code = L.pf_create_with_permeability(C.byref(h), C.byref(self.cfg), _ptr(k))
        else:
            code = L.pf_create(C.byref(h), C.byref(self.cfg))
        _check(code, None)
        self.h = h
        self.info = Info()
        L.pf_get_info(h, C.byref(self.info))
        self.n_lambda = self.info.n_lambda
        n_own = L.pf_owned_subdomains(h, None)
        own = np.zeros(n_own, np.int32)
        L.pf_owned_subdomains(h, _ptr(own))
        self.owned = own.tolist()
        self.subs = []
        for s in self.owned:
            si = SubInfo()
            L.pf_get_sub_info(h, s, C.byref(si))
            self.subs.append({k: getattr(si, k) for k, _ in SubInfo._fields_})

    def close(self):
        if getattr(self, "h", None):
            lib().pf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- reference FetiOperator surface ---
    def apply(self, x):
        x = _vec(x, self.n_lambda, "apply")
        y = np.empty(self.n_lambda)
        _check(lib().pf_apply(self.h, _ptr(x), _ptr(y)), self.h)
        return y

    def apply_preconditioner(self, r):
        r = _vec(r, self.n_lambda, "apply_preconditioner")
        z = np.empty(self.n_lambda)
        _check(lib().pf_apply_precond(self.h, _ptr(r), _ptr(z)), self.h)
        return z

    def project(self, x):
        y = _vec(x, self.n_lambda, "project", copy=True)
        _check(lib().pf_project(self.h, _ptr(y)), self.h)
        return y

    def local_solve(self, s, b):
        if s not in self.owned:
            raise ConfigError(f"local_solve: subdomain {s} is not owned by this engine")
        x = _vec(b, self.subs[self.owned.index(s)]["dim"], "local_solve", copy=True)
        _check(lib().pf_local_solve(self.h, s, _ptr(x)), self.h)
        return x

    def interface_rhs(self):
        F = np.empty(self.n_lambda)
        _check(lib().pf_interface_rhs(self.h, _ptr(F)), self.h)
        return F

    def setup_phases(self):
        """{phase: seconds} of pf_create (setup breakdown)"""
        buf = C.create_string_buffer(4096)
        secs = np.zeros(32)
        n = lib().pf_setup_phases(self.h, buf, 4096, _ptr(secs))
        names = buf.value.decode().split(";") if n > 0 else []
        return {k: float(v) for k, v in zip(names, secs[:n])}

    def set_precond(self, kind):
        """FetiOperator::set_precond (feti.hpp:97): a PRECONDS name."""
        _check(lib().pf_set_precond(self.h, PRECONDS[kind]), self.h)

    def krylov(self, rhs, lambda0, tol, max_iter):
        """feti_pcg (feti.hpp:263-308) on a caller right-hand side -> (lambda,
        report); report["residual_history"] as in REF's PcgReport.  Raises
        SolverError when max_iter is reached (like StepSolver::advance)."""
        rhs = _vec(rhs, self.n_lambda, "krylov: rhs")
        lam = _vec(lambda0, self.n_lambda, "krylov: lambda0", copy=True)
        rep = Report()
        code = lib().pf_krylov(self.h, _ptr(rhs), _ptr(lam), float(tol), int(max_iter), _ptr(lam), C.byref(rep))
        _check(code, self.h)
        d = rep.as_dict()
        d["residual_history"] = self.history()
        return lam, d

    def history(self):
        """residual history of the last Krylov solve (pf_last_history)"""
        n = lib().pf_last_history(self.h, None, 0)
        if n < 0:
            _check(-n, self.h)
        h = np.empty(n)
        lib().pf_last_history(self.h, _ptr(h), n)
        return h

    def back_substitute(self, lam):
        """FetiOperator::back_substitute (feti.hpp:158) for the current
        right-hand side: all owned subdomains' saddle vectors, concatenated."""
        lam = _vec(lam, self.n_lambda, "back_substitute: lambda")
        x = np.empty(self.info.total_dim)
        _check(lib().pf_back_substitute(self.h, _ptr(lam), _ptr(x)), self.h)
        return x

    FIELDS = {"u": 0, "eta": 1, "xi": 2, "p": 3}

    def field(self, name, s=-1):
        """one named field (state.hpp:8-12) of subdomain s, or of every owned
        subdomain concatenated (s = -1)"""
        f = self.FIELDS[name]
        n = lib().pf_field_size(self.h, f, s)
        if n < 0 or (n == 0 and s >= 0):
            raise ConfigError(f"field {name!r} of subdomain {s}: not available")
        out = np.empty(n)
        _check(lib().pf_get_field(self.h, f, s, _ptr(out)), self.h)
        return out

    def constraints(self, s):
        """(saddle index, component (-1: pressure), xy) of subdomain s's essential dofs"""
        n = lib().pf_get_constraints(self.h, s, None, None, None)
        if n < 0:
            raise ConfigError(f"constraints of subdomain {s}: not owned")
        idx, comp, xy = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(2 * n)
        lib().pf_get_constraints(self.h, s, _ptr(idx), _ptr(comp), _ptr(xy))
        return idx, comp, xy.reshape(n, 2)

    def load_sizes(self):
        a, b, c = C.c_longlong(), C.c_longlong(), C.c_longlong()
        _check(lib().pf_load_sizes(self.h, C.byref(a), C.byref(b), C.byref(c)), self.h)
        return a.value, b.value, c.value

    def scenario_loads(self, t):
        """(F_u, Z, g) of the scenario at time t (assemble_loads + constraint values)"""
        nF, nZ, nG = self.load_sizes()
        F, Z, g = np.empty(max(nF, 1)), np.empty(max(nZ, 1)), np.empty(max(nG, 1))
        _check(lib().pf_scenario_loads(self.h, float(t), _ptr(F), _ptr(Z), _ptr(g)), self.h)
        return F[:nF], Z[:nZ], g[:nG]

    def set_loads(self, F_u=None, Z=None, g=None, persistent=False):
        """caller-supplied loads for the next step (every step with persistent)"""
        nF, nZ, nG = self.load_sizes()
        a = None if F_u is None else _vec(F_u, nF, "set_loads: F_u")
        b = None if Z is None else _vec(Z, nZ, "set_loads: Z")
        c = None if g is None else _vec(g, nG, "set_loads: g")
        _check(lib().pf_set_loads(self.h, None if a is None else _ptr(a), None if b is None else _ptr(b),
                                  None if c is None else _ptr(c), int(persistent)), self.h)

    def clear_loads(self):
        _check(lib().pf_clear_loads(self.h), self.h)

    # --- state (StateSnapshot, state.hpp:8-12) ---
    def set_reducer(self, fn):
        """Host reducer for sharded runs: fn(np.ndarray) -> None, sums in place over ranks."""
        proto = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_void_p)

        def cb(user, buf, n, stream):
            fn(np.ctypeslib.as_array(buf, shape=(n,)))

        self._reducer = proto(cb)  # keep alive
        _check(lib().pf_set_reducer(self.h, C.cast(self._reducer, C.c_void_p), None), self.h)

    def state(self):
        xs = []
        for s, S in zip(self.owned, self.subs):
            x = np.empty(S["dim"])
            _check(lib().pf_get_state(self.h, s, _ptr(x)), self.h)
            xs.append(x)
        lam = np.empty(self.n_lambda)
        _check(lib().pf_get_lambda(self.h, _ptr(lam)), self.h)
        return xs, lam

    def errors(self):
        """(err_u, err_p): L2 errors of the current state against the exact
        solution, snapshot_u_error / snapshot_p_error (verify.hpp:62-74),
        computed on the device."""
        eu, ep = C.c_double(), C.c_double()
        _check(lib().pf_errors(self.h, C.byref(eu), C.byref(ep)), self.h)
        return eu.value, ep.value

    def pressure_range(self):
        """(min, max) nodal Darcy pressure of the current state (device)."""
        lo, hi = C.c_double(), C.c_double()
        _check(lib().pf_pressure_range(self.h, C.byref(lo), C.byref(hi)), self.h)
        return lo.value, hi.value

    def write_vtk(self, path):
        """write_solution_vtk (io.hpp:48-86) of the current state."""
        xs, _ = self.state()
        kw = {k: getattr(self.cfg, k) for k in ("mesh_n", "SX", "SY")}
        write_solution_vtk(kw, self.subs, xs, lib().pf_current_step(self.h), path, ids=self.owned)

    def fields(self, xs):
        out = []
        for S, x in zip(self.subs, xs):
            f = {"u": x[:S["n_u"]], "xi": x[S["off_xi"]:S["off_xi"] + S["n_s"]]}
            if S["region"] == 0:
                f["eta"] = x[S["off_eta"]:S["off_eta"] + S["n_s"]]
                f["p"] = x[S["off_p"]:S["off_p"] + S["n_s"]]
            out.append(f)
        return out

    def step(self):
        rep = Report()
        _check(lib().pf_step(self.h, C.byref(rep)), self.h)
        return rep.as_dict()

    def bench_steps(self, nsteps):
        ms = C.c_double()
        it, fa = C.c_int(), C.c_int()
        _check(lib().pf_bench_steps(self.h, nsteps, C.byref(ms), C.byref(it), C.byref(fa)), self.h)
        return ms.value, it.value, fa.value

    def wide_check(self):
        """tests: wide vs scalar per-step sweep on the current right-hand side,
        (differing entries, max |diff|) per elimination-tree level"""
        out = np.zeros(2 * 64)
        n = lib().pf_debug_wide_check(self.h, _ptr(out), 64)
        if n < 0:
            _check(-n, self.h)
        return out[:2 * n].reshape(n, 2)

    def bench(self, kind=0, warmup=5, iters=20):
        ms = C.c_double()
        _check(lib().pf_bench_op(self.h, kind, warmup, iters, C.byref(ms)), self.h)
        sweep, launches = C.c_double(), C.c_int()
        lib().pf_kernel_stats(self.h, C.byref(sweep), C.byref(launches))
        return ms.value, sweep.value, launches.value


def launch_count():
    """Kernels launched by the engine library so far (process-wide)."""
    return int(lib().pf_launch_count())


def phase_stats(op, iters=5):
    out = np.zeros(10)
    _check(lib().pf_phase_stats(op.h, iters, _ptr(out)), op.h)
    return dict(K=out[0:3].tolist(), II=out[3:6].tolist(), Q=out[6:9].tolist(), precond=float(out[9]))


def nccl_unique_id():
    buf = C.create_string_buffer(128)
    _check(lib().pf_nccl_unique_id(buf))
    return buf.raw


def shard_plan(n_sub, rank, nranks):
    """Subdomains owned by `rank` of `nranks` (host-side plan of pf_create_sharded)."""
    out = np.zeros(n_sub, np.int32)
    k = lib().pf_shard_plan(n_sub, rank, nranks, _ptr(out))
    return out[:k].tolist()


class StepSolver:
    """StepSolver (timeloop.hpp:135-193): advance() = one backward-Euler step."""

    def __init__(self, op: FetiOperator):
        self.op = op

    def advance(self, prev_x=None, prev_lambda=None, prev_step=None, out_x=None, out_lambda=None):
        """With no arguments: advance the device-resident state.  With host
        buffers (the reference signature): set the state, step, return the
        next (x_cat, lambda, report).  out_x / out_lambda: caller-owned
        (e.g. page-locked) result buffers."""
        if prev_x is None:
            return self.op.step()
        op = self.op
        x = _vec(prev_x, op.info.total_dim, "advance: prev_x")
        lam = _vec(prev_lambda, op.n_lambda, "advance: prev_lambda")
        nx = np.empty(op.info.total_dim) if out_x is None else out_x
        nl = np.empty(op.n_lambda) if out_lambda is None else out_lambda
        if nx.dtype != np.float64 or not nx.flags.c_contiguous or nx.size != op.info.total_dim:
            raise ConfigError("advance: out_x must be a contiguous float64 array of total_dim")
        if nl.dtype != np.float64 or not nl.flags.c_contiguous or nl.size != op.n_lambda:
            raise ConfigError("advance: out_lambda must be a contiguous float64 array of n_lambda")
        rep = Report()
        _check(lib().pf_advance(op.h, _ptr(x), _ptr(lam), int(prev_step), _ptr(nx), _ptr(nl), C.byref(rep)), op.h)
        return nx, nl, rep.as_dict()


def feti_pcg(op: FetiOperator, rhs, lambda_init, tol, max_iter):
    """feti_pcg (feti.hpp:263): (lambda, report) -- FetiOperator.krylov"""
    return op.krylov(rhs, lambda_init, tol, max_iter)


def unpack_state(op: FetiOperator):
    """unpack_state (feti.hpp:443-454) of the device-resident state into the
    reference's StateSnapshot names.  One poroelastic and one elastic
    subdomain (the reference layout): u_P, eta, xi_P, p, u_E, xi_E, lambda;
    otherwise per-region fields concatenated over the subdomains of that region
    in subdomain order."""
    P = [s for s, S in zip(op.owned, op.subs) if S["region"] == 0]
    E = [s for s, S in zip(op.owned, op.subs) if S["region"] != 0]
    cat = lambda name, ids: np.concatenate([op.field(name, s) for s in ids]) if ids else np.empty(0)
    _, lam = op.state()
    return {"step": lib().pf_current_step(op.h), "u_P": cat("u", P), "eta": cat("eta", P), "xi_P": cat("xi", P),
            "p": cat("p", P), "u_E": cat("u", E), "xi_E": cat("xi", E), "lambda": lam}


def local_matrices(tri, mu, order, kperm=1.0, mu_f=1.0):
    """local_elastic_matrix / local_div_matrix / local_mass_matrix /
    local_diffusion_matrix (elements.hpp:152-230) of one triangle, on the device"""
    tri = np.ascontiguousarray(tri, np.float64).reshape(6)
    nb = 3 if order == 1 else 6
    el, dv = np.empty((2 * nb, 2 * nb)), np.empty((3, 2 * nb))
    ma, di = np.empty((3, 3)), np.empty((3, 3))
    _check(lib().pf_local_matrices(_ptr(tri), float(mu), float(kperm), float(mu_f), int(order), _ptr(el), _ptr(dv),
                                   _ptr(ma), _ptr(di)))
    return {"elastic": el, "div": dv, "mass": ma, "diffusion": di}


def run_simulation(op: FetiOperator, steps=None):
    """run_simulation (timeloop.hpp:206-221): all steps, returns the reports."""
    n = op.info.N if steps is None else steps
    return [op.step() for _ in range(n)]


class PinnedArray(np.ndarray):
    """float64 array in page-locked host memory (pf_host_alloc), freed with
    the last view."""

    def __array_finalize__(self, obj):
        if obj is not None and not hasattr(self, "_pin"):
            self._pin = getattr(obj, "_pin", None)


class _Pin:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().pf_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(n):
    """np.empty(n) in page-locked memory (for StepSolver.advance host buffers)."""
    p = C.c_void_p()
    _check(lib().pf_host_alloc(8 * max(int(n), 1), C.byref(p)))
    buf = (C.c_double * max(int(n), 1)).from_address(p.value)
    a = np.frombuffer(buf, dtype=np.float64, count=int(n)).view(PinnedArray)
    a._pin = _Pin(p.value)
    return a


def oscillation_check(ranges, max_boundary, delta):
    """oscillation_check (verify.hpp:167-195) on per-snapshot nodal pressure
    ranges [(min, max), ...] (FetiOperator.pressure_range after each step):
    the pressure must stay within [-delta, max_boundary + delta]; the worst
    offender is reported."""
    rep = {"pass": True, "lower_bound": -delta, "upper_bound": max_boundary + delta, "worst_violation": 0.0}
    lo = min((r[0] for r in ranges), default=float("inf"))
    hi = max((r[1] for r in ranges), default=float("-inf"))
    if not np.isfinite(lo):
        lo = hi = 0.0
    rep["min_p"], rep["max_p"] = lo, hi
    worst = 0.0
    if lo < rep["lower_bound"] and rep["lower_bound"] - lo > worst:
        worst = rep["lower_bound"] - lo
        rep["worst_violation"], rep["pass"] = lo, False
    if hi > rep["upper_bound"] and hi - rep["upper_bound"] > worst:
        rep["worst_violation"], rep["pass"] = hi, False
    return rep


def barry_mercer_check(mesh_n=16, order=2, dt=1e-2, T=None, bound_frac=0.05, E=1e4, nu=0.2, c0=0.1, **kw):
    """The paper's Barry-Mercer oscillation study (model.hpp:274-324 +
    verify.hpp:160-195; h = 1/16, tau = 1e-2, bound 0.05 max|p2|)
    on the device: runs the reference layout, reads the nodal pressure range
    after every step (pf_pressure_range, no state download) and applies
    oscillation_check with max_boundary = max_t |sin t| over the steps."""
    import math
    steps = max(1, int(round((T if T is not None else 10 * dt) / dt)))
    op = FetiOperator(**dict(dict(mesh_n=mesh_n, SX=1, SY=2, order=order, scenario="barry-mercer", E=E, nu=nu,
                                  c0=c0, dt=dt, steps=steps, precond="dirichlet"), **kw))
    try:
        ranges = []
        for _ in range(steps):
            op.step()
            ranges.append(op.pressure_range())
    finally:
        op.close()
    max_bnd = max(abs(math.sin(k * dt)) for k in range(1, steps + 1))
    return oscillation_check(ranges, max_bnd, bound_frac * max_bnd)


def estimate_order(err_coarse, err_fine, h_coarse, h_fine):
    """verify.hpp:85-87."""
    return float(np.log(err_coarse / err_fine) / np.log(h_coarse / h_fine))


def mms_errors(nu, mesh_n, fe_order=2, E=1e4, T=1e-2, dt=1e-3, mu_conv="paper", **kw):
    """mms_errors (verify.hpp:108-123) on the device: one manufactured-solution
    run of the reference layout (reference `mms` scenario unless `scenario` is
    given), L-inf over the snapshots (steps 1..N, timeloop.hpp:206-221) of the
    spatial L2 errors of u and p."""
    steps = max(1, int(round(T / dt)))
    cfg = dict(dict(mesh_n=mesh_n, SX=1, SY=2, order=fe_order, E=E, nu=nu, dt=dt, steps=steps, scenario="mms",
                    precond="dirichlet", mu_conv=mu_conv, c0=0.1), **kw)
    op = FetiOperator(**cfg)
    try:
        eu = ep = 0.0
        for _ in range(steps):
            op.step()
            u, p = op.errors()
            eu, ep = max(eu, u), max(ep, p)
        return eu, ep
    finally:
        op.close()


def convergence_study(mesh_sizes=(8, 16, 24, 32), nus=(0.2, 0.49, 0.499, 0.4999), fe_order=2, E=1e4, T=1e-2,
                      dt=1e-3, mu_conv="paper", verbose=False, **kw):
    """convergence_study (verify.hpp:125-158): rows (nu, h, err_u, order_u,
    err_p, order_p) per (nu, mesh); a failed run drops its row and the study
    continues (the order chain restarts)."""
    rows = []
    for nu in nus:
        prev = None
        for n in mesh_sizes:
            h = 1.0 / n
            try:
                eu, ep = mms_errors(nu, n, fe_order, E, T, dt, mu_conv, **kw)
            except Error as e:
                import sys
                print(f"convergence_study: run nu={nu:g} n={n} failed: {e}", file=sys.stderr)
                prev = None
                continue
            row = {"nu": nu, "h": h, "err_u": eu, "order_u": float("nan"), "err_p": ep, "order_p": float("nan")}
            if prev is not None:
                row["order_u"] = estimate_order(prev["err_u"], eu, prev["h"], h)
                row["order_p"] = estimate_order(prev["err_p"], ep, prev["h"], h)
            if verbose:
                print(f"nu={nu:<7g} h=1/{n:<3d}  err_u={eu:.6e} ord_u={row['order_u']:6.3f}  "
                      f"err_p={ep:.6e} ord_p={row['order_p']:6.3f}")
            rows.append(row)
            prev = row
    return rows


def _num(v):
    """detail::num (io.hpp:23-27): %.12g."""
    return "%.12g" % v


def write_error_csv(rows, path):
    """write_error_table_csv (io.hpp:96-106): header nu,h,err_u,order_u,err_p,order_p
    (SPEC.md:527); non-finite orders (the first row of each nu) left empty."""
    import math
    with open(path, "w") as f:
        f.write("nu,h,err_u,order_u,err_p,order_p\n")
        for r in rows:
            ou = _num(r["order_u"]) if math.isfinite(r["order_u"]) else ""
            op = _num(r["order_p"]) if math.isfinite(r["order_p"]) else ""
            f.write(f"{_num(r['nu'])},{_num(r['h'])},{_num(r['err_u'])},{ou},{_num(r['err_p'])},{op}\n")


VARIANT_NAMES = {"generalized": "feti-generalized", "dirichlet": "feti-schur",
                 "generalized-mortar": "feti-generalized-mortar", "dirichlet-mortar": "feti-schur-mortar",
                 "identity": "feti-identity"}


def write_solver_log_csv(reports, path, precond="dirichlet"):
    """write_solver_log_csv (io.hpp:108-114): step,variant,iterations,residual,
    time_p,time_e per step report.  The reference's time_P / time_E are the
    seconds of its two subdomain solves; here every subdomain runs in one
    launch, so time_p carries the step's device seconds and time_e 0."""
    with open(path, "w") as f:
        f.write("step,variant,iterations,residual,time_p,time_e\n")
        for r in reports:
            f.write(f"{r['step']},{VARIANT_NAMES.get(precond, precond)},{r['iterations']},"
                    f"{_num(r['rel_residual'])},{_num(r['seconds'])},{_num(0.0)}\n")


def write_solution_vtk(cfg, subs, xs, step, path, ids=None):
    """write_solution_vtk (io.hpp:48-86) for a partition: every subdomain's
    triangulation appended (vertices row-major bottom to top, cells split
    (a,b,c),(a,c,d), mesh.hpp:104-131), point data subsampled to the vertices
    (P2 midside values dropped); displacement on every point, pressure and
    fluid content zero on elastic points, elastic pressure xi on both.
    cfg: make_config keywords; subs: per-subdomain info (region, n_u, n_s,
    off_eta, off_xi, off_p) in subdomain order s = sy*SX + sx; xs: the
    subdomains' saddle vectors (FetiOperator.state or the oracle's); ids: their
    subdomain indices (default 0..len-1; a shard passes its owned list)."""
    n, SX, SY = int(cfg["mesh_n"]), int(cfg["SX"]), int(cfg["SY"])
    cx, cy = n // SX, n // SY
    nvs = (cx + 1) * (cy + 1)
    pts, cells, disp, pres, xi, eta = [], [], [], [], [], []
    for k, (S, x) in enumerate(zip(subs, xs)):
        s = ids[k] if ids is not None else k
        sx, sy = s % SX, s // SX
        base = len(pts)
        for j in range(cy + 1):
            for i in range(cx + 1):
                pts.append(((sx * cx + i) / n, (sy * cy + j) / n))
        for j in range(cy):
            for i in range(cx):
                a = base + j * (cx + 1) + i
                b, c, d = a + 1, a + cx + 2, a + cx + 1
                cells += [(a, b, c), (a, c, d)]
        u = x[:S["n_u"]]
        disp += [(u[2 * v], u[2 * v + 1]) for v in range(nvs)]
        xi += list(x[S["off_xi"]:S["off_xi"] + nvs])
        P = S["region"] == 0
        pres += list(x[S["off_p"]:S["off_p"] + nvs]) if P else [0.0] * nvs
        eta += list(x[S["off_eta"]:S["off_eta"] + nvs]) if P else [0.0] * nvs
    with open(path, "w") as f:
        f.write(f"# vtk DataFile Version 3.0\nporofeti solution step {step}\nASCII\nDATASET UNSTRUCTURED_GRID\n")
        f.write(f"POINTS {len(pts)} double\n")
        f.writelines(f"{_num(px)} {_num(py)} 0\n" for px, py in pts)
        f.write(f"CELLS {len(cells)} {4 * len(cells)}\n")
        f.writelines(f"3 {a} {b} {c}\n" for a, b, c in cells)
        f.write(f"CELL_TYPES {len(cells)}\n" + "5\n" * len(cells))
        f.write(f"POINT_DATA {len(pts)}\nVECTORS displacement double\n")
        f.writelines(f"{_num(ux)} {_num(uy)} 0\n" for ux, uy in disp)
        for name, vals in (("pressure", pres), ("elastic_pressure", xi), ("fluid_content", eta)):
            f.write(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
            f.writelines(f"{_num(v)}\n" for v in vals)


def debug_factor_solve(A, ic, b, mode=1, task_cap=4096):
    """Host-logic check of the symbolic layout (CPU): solve A x = b with the
    engine's ordering/supernodes/task schedule emulated on the host."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    ptr = np.ascontiguousarray(A.indptr, np.int32)
    col = np.ascontiguousarray(A.indices, np.int32)
    val = np.ascontiguousarray(A.data, np.float64)
    icc = np.ascontiguousarray(ic, np.int32).reshape(-1)
    x = np.array(b, np.float64)
    stats = np.zeros(6, np.int64)
    _check(lib().pf_debug_factor_solve(n, _ptr(ptr), _ptr(col), _ptr(val), _ptr(icc), _ptr(x), mode, task_cap,
                                       _ptr(stats)))
    return x, stats


def debug_disc(config: Config, s=0):
    sizes = np.zeros(5, np.int64)
    nG, nK = C.c_int(), C.c_int()
    _check(lib().pf_debug_disc(C.byref(config), _ptr(sizes), s, C.byref(nG), None, None, None, C.byref(nK), None,
                               None, None))
    gl = np.zeros(max(nG.value, 1), np.int32)
    gc = np.zeros(max(nG.value, 1), np.int32)
    gv = np.zeros(max(nG.value, 1))
    dim = None
    kp = None
    # K pattern: rows = dim of subdomain s; allocate generously
    kc = np.zeros(max(nK.value, 1), np.int32)
    kp = np.zeros(int(sizes[4]) + 1, np.int32)
    ic = np.zeros(2 * int(sizes[4]), np.int32)
    _check(lib().pf_debug_disc(C.byref(config), _ptr(sizes), s, C.byref(nG), _ptr(gl), _ptr(gc), _ptr(gv),
                               C.byref(nK), _ptr(kp), _ptr(kc), _ptr(ic)))
    return dict(n_sub=int(sizes[0]), n_lambda=int(sizes[1]), n_lambda_u=int(sizes[2]), n_types=int(sizes[3]),
                total_dim=int(sizes[4]), G=(gl[:nG.value], gc[:nG.value], gv[:nG.value]), K_ptr=kp,
                K_col=kc[:nK.value], dof_ic=ic)
