"""ctypes wrapper of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the checker.  The product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "_build", "liboracle.so")

SCENARIOS = {"mms-t": 0, "mms": 1, "injection": 2, "barry-mercer": 3}
PRECONDS = {"identity": 0, "generalized": 1, "dirichlet": 2, "generalized-mortar": 3, "dirichlet-mortar": 4}
KRYLOV = {"auto": 0, "pcg": 1, "minres": 2, "sqmr": 3}


class Config(C.Structure):
    """Mirror of or_config / pf_config (same field order in both C headers)."""

    _fields_ = [
        ("mesh_n", C.c_int), ("SX", C.c_int), ("SY", C.c_int), ("order", C.c_int),
        ("E", C.c_double), ("nu", C.c_double), ("alpha", C.c_double), ("c0", C.c_double),
        ("kperm", C.c_double), ("mu_f", C.c_double), ("dt", C.c_double),
        ("steps", C.c_int), ("mu_conv", C.c_int), ("scenario", C.c_int),
        ("precond", C.c_int), ("krylov", C.c_int),
        ("tol", C.c_double), ("max_iter", C.c_int), ("warm", C.c_int), ("threads", C.c_int),
        ("seed", C.c_ulonglong), ("logk_mean", C.c_double), ("logk_sd", C.c_double),
    ]


def make_config(mesh_n=32, SX=1, SY=2, order=1, E=1.0, nu=0.3, alpha=1.0, c0=1e-3, kperm=1.0,
                mu_f=1.0, dt=1e-2, steps=5, mu_conv="paper", scenario="mms-t", precond="dirichlet",
                krylov="auto", tol=1e-10, max_iter=500, warm=True, threads=0, seed=20240901,
                logk_mean=-2.0, logk_sd=1.0, cls=Config):
    return cls(mesh_n, SX, SY, order, E, nu, alpha, c0, kperm, mu_f, dt, steps,
               0 if mu_conv == "paper" else 1, SCENARIOS[scenario], PRECONDS[precond],
               KRYLOV[krylov], tol, max_iter, int(warm), threads, seed, logk_mean, logk_sd)


# BASELINE.json configs (c1..c5); steps/dt as stated there.
BASELINE_CONFIGS = {
    "c1": dict(mesh_n=32, SX=1, SY=2, order=1, nu=0.3, c0=1e-3, dt=1e-2, steps=5, scenario="mms-t"),
    "c2": dict(mesh_n=128, SX=2, SY=2, order=2, nu=0.3, c0=1e-3, dt=1e-2, steps=10, scenario="mms-t"),
    "c3": dict(mesh_n=512, SX=8, SY=8, order=2, nu=0.49999, c0=1e-3, dt=1e-3, steps=20, scenario="mms-t",
               max_iter=3000),
    "c4": dict(mesh_n=1024, SX=32, SY=32, order=2, nu=0.3, c0=1e-3, dt=1e-2, steps=10, scenario="mms-t"),
    "c5": dict(mesh_n=512, SX=16, SY=16, order=2, nu=0.4, c0=1e-4, dt=1e-3, steps=100,
               scenario="injection", max_iter=3000),
}


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        L.or_last_error.restype = C.c_char_p
        L.or_create.argtypes = [C.POINTER(Config), C.POINTER(P)]
        L.or_destroy.argtypes = [P]
        L.or_info.argtypes = [P, ip, dp]
        L.or_sub_info.argtypes = [P, C.c_int, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
        L.or_sub_matrix.argtypes = [P, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_apply.argtypes = [P, dp, dp]
        L.or_precond.argtypes = [P, dp, dp]
        L.or_project.argtypes = [P, dp]
        L.or_local_solve.argtypes = [P, C.c_int, dp]
        L.or_step_rhs.argtypes = [P, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_run.argtypes = [P, C.c_int]
        L.or_n_states.argtypes = [P]
        L.or_state.argtypes = [P, C.c_int, C.c_int, dp]
        L.or_lambda.argtypes = [P, C.c_int, dp]
        L.or_errors.argtypes = [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.or_report.argtypes = [P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p,
                                C.POINTER(C.c_int)]
        L.or_report_true.argtypes = [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.or_monolithic_step.argtypes = [P, dp, dp]
        L.or_mults.argtypes = [P, ip, C.c_void_p]
        L.or_n_ifaces.argtypes = [P]
        L.or_kelem.argtypes = [P, dp]
        L.or_n_src.argtypes = [P]
        L.or_apply_subset.argtypes = [P, dp, dp, ip, C.c_int, C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(code):
    if code != 0:
        raise OracleError(code, lib().or_last_error().decode())


class Oracle:
    """One oracle discretisation + factorised FETI operator."""

    def __init__(self, **kw):
        self.cfg = make_config(**kw)
        L = lib()
        h = C.c_void_p()
        check(L.or_create(C.byref(self.cfg), C.byref(h)))
        self.h = h
        info = np.zeros(7, np.int32)
        dinfo = np.zeros(9)
        L.or_info(h, info, dinfo)
        (self.n_sub, self.n_lambda, self.n_lambda_u, self.n_coarse, self.minres, self.N,
         self.n_floating) = (int(v) for v in info)
        self.tau, self.T, self.t_setup, self.t_factor = dinfo[:4]
        self.lam_P, self.mu_P, self.k1, self.k2, self.k3 = dinfo[4:]
        self.subs = []
        for s in range(self.n_sub):
            si = np.zeros(14, np.int64)
            L.or_sub_info(h, s, si)
            keys = ["region", "dim", "n_u", "n_s", "off_u", "off_eta", "off_xi", "off_p",
                    "floating", "nnzK", "n_cons", "nnzL", "nBu", "nBp"]
            self.subs.append({k: int(v) for k, v in zip(keys, si)})

    def __del__(self):
        try:
            lib().or_destroy(self.h)
        except Exception:
            pass

    def matrix(self, s, which):
        """which: K, G, Gc, lift, A, B, R, Af -> scipy.sparse.csr_matrix"""
        import scipy.sparse as sp
        idx = ["K", "G", "Gc", "lift", "A", "B", "R", "Af"].index(which)
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int()
        L = lib()
        check(L.or_sub_matrix(self.h, s, idx, C.byref(nr), C.byref(nc), C.byref(nnz), None, None, None))
        ptr = np.zeros(nr.value + 1, np.int32)
        col = np.zeros(max(nnz.value, 1), np.int32)
        val = np.zeros(max(nnz.value, 1))
        check(L.or_sub_matrix(self.h, s, idx, C.byref(nr), C.byref(nc), C.byref(nnz),
                              ptr.ctypes.data, col.ctypes.data, val.ctypes.data))
        return sp.csr_matrix((val[:nnz.value], col[:nnz.value], ptr), shape=(nr.value, nc.value))

    def mults(self):
        m = np.zeros(3 * self.n_lambda, np.int32)
        nif = lib().or_n_ifaces(self.h)
        ifs = np.zeros(4 * max(nif, 1), np.int32)
        lib().or_mults(self.h, m, ifs.ctypes.data)
        return m.reshape(-1, 3), ifs[:4 * nif].reshape(-1, 4)

    def apply(self, x):
        y = np.zeros(self.n_lambda)
        check(lib().or_apply(self.h, np.ascontiguousarray(x, np.float64), y))
        return y

    def apply_subset(self, x, subs, which=0):
        y = np.zeros(self.n_lambda)
        s = np.ascontiguousarray(subs, np.int32)
        check(lib().or_apply_subset(self.h, np.ascontiguousarray(x, np.float64), y, s, len(s), which))
        return y

    def precond(self, x):
        y = np.zeros(self.n_lambda)
        check(lib().or_precond(self.h, np.ascontiguousarray(x, np.float64), y))
        return y

    def project(self, x):
        y = np.array(x, np.float64)
        check(lib().or_project(self.h, y))
        return y

    def local_solve(self, s, b):
        x = np.array(b, np.float64)
        check(lib().or_local_solve(self.h, s, x))
        return x

    def step_rhs(self, step=0):
        tot = sum(S["dim"] for S in self.subs)
        b = np.zeros(tot)
        d = np.zeros(self.n_lambda)
        F = np.zeros(self.n_lambda)
        check(lib().or_step_rhs(self.h, step, b.ctypes.data, d.ctypes.data, F.ctypes.data))
        return self.split(b), d, F

    def split(self, cat):
        out, o = [], 0
        for S in self.subs:
            out.append(cat[o:o + S["dim"]])
            o += S["dim"]
        return out

    def run(self, nsteps):
        check(lib().or_run(self.h, nsteps))

    def state(self, step):
        xs = []
        for s, S in enumerate(self.subs):
            x = np.zeros(S["dim"])
            check(lib().or_state(self.h, step, s, x))
            xs.append(x)
        lam = np.zeros(self.n_lambda)
        check(lib().or_lambda(self.h, step, lam))
        return xs, lam

    def errors(self, step):
        """verify.hpp:62-74 on time level `step`: (err_u, err_p)."""
        eu, ep = C.c_double(), C.c_double()
        check(lib().or_errors(self.h, step, C.byref(eu), C.byref(ep)))
        return eu.value, ep.value

    def report(self, step):
        it, conv, nh = C.c_int(), C.c_int(), C.c_int()
        rel, secs = C.c_double(), C.c_double()
        check(lib().or_report(self.h, step, C.byref(it), C.byref(conv), C.byref(rel), C.byref(secs),
                              None, C.byref(nh)))
        hist = np.zeros(nh.value)
        check(lib().or_report(self.h, step, C.byref(it), C.byref(conv), C.byref(rel), C.byref(secs),
                              hist.ctypes.data, C.byref(nh)))
        tr, rs = C.c_double(), C.c_int()
        check(lib().or_report_true(self.h, step, C.byref(tr), C.byref(rs)))
        return dict(iterations=it.value, converged=bool(conv.value), rel_residual=rel.value,
                    seconds=secs.value, history=hist, true_residual=tr.value, restarts=rs.value)

    def monolithic_step(self):
        tot = sum(S["dim"] for S in self.subs)
        x = np.zeros(tot)
        lam = np.zeros(self.n_lambda)
        check(lib().or_monolithic_step(self.h, x, lam))
        return self.split(x), lam

    def kelem(self):
        k = np.zeros(2 * self.cfg.mesh_n ** 2)
        lib().or_kelem(self.h, k)
        return k

    def n_src(self):
        return lib().or_n_src(self.h)

    def fields(self, xs):
        """Split saddle solutions into named fields per subdomain."""
        out = []
        for S, x in zip(self.subs, xs):
            f = {"u": x[S["off_u"]:S["off_u"] + S["n_u"]], "xi": x[S["off_xi"]:S["off_xi"] + S["n_s"]]}
            if S["region"] == 0:
                f["eta"] = x[S["off_eta"]:S["off_eta"] + S["n_s"]]
                f["p"] = x[S["off_p"]:S["off_p"] + S["n_s"]]
            out.append(f)
        return out


# ---------------------------------------------------------------------------
# element / mesh level entry points (re-expression of the reference's own
# known-answer tests, tests/test_elements.cpp and tests/test_mesh.cpp)
# ---------------------------------------------------------------------------
def _kat_lib():
    L = lib()
    if getattr(L, "_kat_ready", False):
        return L
    vp = C.c_void_p
    L.or_triangle_rule.argtypes = [C.c_int, vp, vp, C.POINTER(C.c_int)]
    L.or_edge_rule.argtypes = [C.c_int, vp, vp, C.POINTER(C.c_int)]
    L.or_eval_basis.argtypes = [C.c_int, C.c_double, C.c_double, vp, vp]
    L.or_local_elastic.argtypes = [vp, C.c_double, C.c_int, vp]
    L.or_local_div.argtypes = [vp, C.c_int, vp]
    L.or_local_mass.argtypes = [vp, vp]
    L.or_local_diffusion.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_double, vp]
    L.or_local_interface.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, vp]
    L.or_mesh_build.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.or_mesh_free.argtypes = [vp]
    L.or_mesh_counts.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.or_mesh_vertices.argtypes = [vp, vp]
    L.or_mesh_triangles.argtypes = [vp, vp, vp]
    L.or_mesh_tag.argtypes = [vp, C.c_int, C.c_double]
    L.or_mesh_boundary.argtypes = [vp, vp, vp, vp, vp, vp]
    L.or_dofmap.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), vp]
    L.or_pair.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int), vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L._kat_ready = True
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def triangle_rule(degree):
    pts, w, n = np.zeros(12), np.zeros(6), C.c_int()
    check(_kat_lib().or_triangle_rule(degree, _p(pts), _p(w), C.byref(n)))
    return pts[:2 * n.value].reshape(-1, 2), w[:n.value]


def edge_rule(degree):
    pts, w, n = np.zeros(3), np.zeros(3), C.c_int()
    check(_kat_lib().or_edge_rule(degree, _p(pts), _p(w), C.byref(n)))
    return pts[:n.value], w[:n.value]


def eval_basis(order, x, y):
    v, g = np.zeros(6), np.zeros(12)
    check(_kat_lib().or_eval_basis(order, x, y, _p(v), _p(g)))
    nb = 3 if order == 1 else 6
    return v[:nb], g[:2 * nb].reshape(-1, 2)


def _tri(tri):
    return np.ascontiguousarray(np.asarray(tri, np.float64).reshape(6))


def local_elastic(tri, mu, order):
    nb = 3 if order == 1 else 6
    out = np.zeros((2 * nb, 2 * nb))
    check(_kat_lib().or_local_elastic(_p(_tri(tri)), mu, order, _p(out)))
    return out


def local_div(tri, order):
    nb = 3 if order == 1 else 6
    out = np.zeros((3, 2 * nb))
    check(_kat_lib().or_local_div(_p(_tri(tri)), order, _p(out)))
    return out


def local_mass(tri):
    out = np.zeros((3, 3))
    check(_kat_lib().or_local_mass(_p(_tri(tri)), _p(out)))
    return out


def local_diffusion(tri, K, mu_f):
    out = np.zeros((3, 3))
    check(_kat_lib().or_local_diffusion(_p(_tri(tri)), K[0][0], K[0][1], K[1][1], mu_f, _p(out)))
    return out


def local_interface(a, b, trace_order):
    out = np.zeros((2, trace_order + 1))
    check(_kat_lib().or_local_interface(a[0], a[1], b[0], b[1], trace_order, _p(out)))
    return out


class Mesh:
    """oracle Mesh (mesh.hpp restatement): region 0 = P, 1 = E."""

    def __init__(self, region, rect, nx, ny):
        h = C.c_void_p()
        r = np.asarray(rect, np.float64)
        check(_kat_lib().or_mesh_build(region, _p(r), nx, ny, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            _kat_lib().or_mesh_free(self.h)
        except Exception:
            pass

    def counts(self):
        nv, nt, ne = C.c_int(), C.c_int(), C.c_int()
        _kat_lib().or_mesh_counts(self.h, C.byref(nv), C.byref(nt), C.byref(ne))
        return nv.value, nt.value, ne.value

    def vertices(self):
        nv = self.counts()[0]
        xy = np.zeros(2 * nv)
        _kat_lib().or_mesh_vertices(self.h, _p(xy))
        return xy.reshape(-1, 2)

    def triangles(self):
        nt = self.counts()[1]
        t, a = np.zeros(3 * nt, np.int32), np.zeros(nt)
        _kat_lib().or_mesh_triangles(self.h, _p(t), _p(a))
        return t.reshape(-1, 3), a

    def tag(self, rule, param=0.5):
        check(_kat_lib().or_mesh_tag(self.h, rule, param))

    def boundary(self):
        n = 4 * sum(self.counts())
        e, m, pt, i = (np.zeros(n, np.int32) for _ in range(4))
        mid = np.zeros(2 * n)
        k = _kat_lib().or_mesh_boundary(self.h, _p(e), _p(m), _p(pt), _p(i), _p(mid))
        return e[:k], m[:k], pt[:k], i[:k].astype(bool), mid[:2 * k].reshape(-1, 2)

    def dofmap(self, kind, order):
        nn, nd = C.c_int(), C.c_int()
        on = np.zeros(sum(self.counts()) + 8, np.int8)
        check(_kat_lib().or_dofmap(self.h, kind, order, C.byref(nn), C.byref(nd), _p(on)))
        return nn.value, nd.value, on[:nn.value].astype(bool)


def pair(ma, mb, order):
    npairs, nmult, ned = C.c_int(), C.c_int(), C.c_int()
    pairs = np.zeros(2 * (sum(ma.counts()) + 8), np.int32)
    check(_kat_lib().or_pair(ma.h, mb.h, order, C.byref(npairs), _p(pairs), C.byref(nmult), C.byref(ned)))
    return pairs[:2 * npairs.value].reshape(-1, 2), nmult.value, ned.value
