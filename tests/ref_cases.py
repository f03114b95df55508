"""The reference-run fixtures tests/golden/ref_<case>.npz (made by
oracle/ref/make_ref_golden.py from the UNMODIFIED reference compiled against
the Eigen-API shim) and the equivalent configurations of the oracle and the
engine.  Shared by tests/test_ref_pin.py (oracle, CPU) and
tests/test_gpu_ref_pin.py (engine, GPU)."""
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
C1 = dict(mesh_n=32, SX=1, SY=2, order=1, nu=0.3, c0=1e-3, dt=1e-2, scenario="mms-t")
REF_DEFAULT = dict(SX=1, SY=2, order=2, E=1e4, nu=0.2, c0=0.1)  # model.hpp:92-95 default_params
CASES = {
    "c1_schur": dict(C1, steps=5, precond="dirichlet"),
    "c1_generalized": dict(C1, steps=5, precond="generalized"),
    "mms_m8": dict(REF_DEFAULT, mesh_n=8, dt=1e-4, steps=2, scenario="mms", precond="dirichlet"),
    "mms_m16": dict(REF_DEFAULT, mesh_n=16, dt=1e-4, steps=2, scenario="mms", precond="dirichlet"),
    "mms_m32": dict(REF_DEFAULT, mesh_n=32, dt=1e-4, steps=2, scenario="mms", precond="dirichlet"),
    "bm_m8": dict(REF_DEFAULT, mesh_n=8, dt=1e-2, steps=3, scenario="barry-mercer", precond="dirichlet"),
    "bm_m16": dict(REF_DEFAULT, mesh_n=16, dt=1e-2, steps=3, scenario="barry-mercer", precond="dirichlet"),
    "bm_m32": dict(REF_DEFAULT, mesh_n=32, dt=1e-2, steps=3, scenario="barry-mercer", precond="dirichlet"),
}
FIELDS = ("u_P", "eta", "xi_P", "p", "u_E", "xi_E", "lambda")


def load(name):
    return np.load(os.path.join(GOLD, f"ref_{name}.npz"))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def named_fields(fields_P, fields_E, lam):
    """oracle / engine per-subdomain fields -> the reference's StateSnapshot names (state.hpp:8-12)"""
    return {"u_P": fields_P["u"], "eta": fields_P["eta"], "xi_P": fields_P["xi"], "p": fields_P["p"],
            "u_E": fields_E["u"], "xi_E": fields_E["xi"], "lambda": lam}


def field_bar(z, k, f, floor):
    """max(floor, 10x the reference's own spread): the spread is how far the
    reference moves between two equally valid elimination orders of its LU
    (EIGEN_SHIM_ORDER=rcm vs cm), i.e. the rounding floor of the reference's
    answer at this tolerance."""
    return max(floor, 10.0 * float(z[f"spread_{f}{k}"]))


def ill_conditioned(name):
    """E = 1e4 cases: the local saddles reach cond ~ 1e11 (mesh 8); the
    reference's LU solves make F nonsymmetric at 1e-12..1e-10 (measured,
    DESIGN.md) which slows its PCG tail; LDL^T-based solves (oracle, engine)
    are symmetric to 1e-16 and need no more iterations."""
    return not name.startswith("c1")


def iteration_window(hist, tol):
    """+-2 around the count of a run with residual history `hist`, widened to
    its noise plateau (iterations already within 10x of the tolerance)."""
    h = np.asarray(hist) / hist[0]
    k = len(h) - 1
    near = [j for j in range(len(h)) if h[j] <= 10.0 * tol]
    lo = min([k - 2] + near)
    return lo, k + max(2, k - lo)
