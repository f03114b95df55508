"""The direct interface solve (krylov="direct"): the GPU analogue of the
reference's monolithic solver (SolverChoice::monolithic, feti.hpp:313-440,
timeloop.hpp:139-160).

The coupled system is condensed exactly onto the multipliers, the interface
operator F is assembled dense from the explicit local operators and inverted
once (signed Cholesky on the FP64 tensor cores; bordered by the rigid-mode
constraint of the floating subdomains), and every step is one GEMV plus the
same back-substitution as the FETI path.  Checked against
  * the reference's OWN monolithic run of BASELINE config 1 (all 5 steps);
  * the oracle's monolithic restatement (dense LU of the whole coupled system)
    on multi-subdomain layouts with floating subdomains, pressure multipliers,
    nu = 0.49999 and the heterogeneous injection permeability;
  * the oracle's FETI solution at a tight Krylov tolerance at BASELINE c2's
    full size, and the full-size c3 / c5 fixtures.
"""
import os

import numpy as np
import pytest

import paper_2509_06673_b200 as pf
from ref_cases import CASES, FIELDS, load, named_fields, rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_direct_c1_matches_reference_monolithic():
    """BASELINE c1 through the direct path vs the reference's own MonolithicSolver
    (Eigen-API shim build, tests/golden/ref_c1_monolithic.npz): every field of
    all 5 steps within 1e-10 (both are direct solves of the same system)."""
    z = load("c1_monolithic")
    kw = dict(CASES["c1_schur"], krylov="direct")
    op = pf.FetiOperator(**kw)
    assert op.info.krylov == 4
    for k in range(1, 6):
        rep = op.step()
        assert rep["converged"] and rep["iterations"] == 0 and rep["method"] == "direct"
        assert rep["true_residual"] <= 1e-12, rep
        xs, lam = op.state()
        f = op.fields(xs)
        got = named_fields(f[0], f[1], lam)
        for fld in FIELDS:
            ref = z[f"{fld}{k}"]
            if np.linalg.norm(ref) == 0:
                continue
            bar = max(1e-10, 10.0 * float(z[f"spread_{fld}{k}"]))
            assert rel(got[fld], ref) <= bar, (k, fld, rel(got[fld], ref), bar)
    op.close()


SMALL = {
    # 4x4 subdomains of 4x4 P2 cells: 4 floating, P|P pressure multipliers
    "c4_params": dict(pf.BASELINE_CONFIGS["c4"], mesh_n=16, SX=4, SY=4, steps=1),
    "c3_params": dict(pf.BASELINE_CONFIGS["c3"], mesh_n=16, SX=4, SY=4, steps=1),
    "c5_params": dict(pf.BASELINE_CONFIGS["c5"], mesh_n=16, SX=4, SY=4, steps=1),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_direct_matches_oracle_monolithic(name):
    """Step 1 vs the oracle's dense LU of the whole coupled system
    [blockdiag(K_s) G^T; G 0] (o_feti.hpp monolithic_solve): u, xi, eta, p and
    lambda within 1e-8 relative L2 per subdomain field."""
    import oracle_lib as ol
    kw = dict(SMALL[name], krylov="direct")
    op = pf.FetiOperator(**kw)
    assert op.info.n_coarse > 0 and op.n_lambda > op.info.n_lambda_u
    rep = op.step()
    assert rep["iterations"] == 0 and rep["true_residual"] <= 1e-11, rep
    xs, lam = op.state()
    o = ol.Oracle(**SMALL[name])
    xo, lo = o.monolithic_step()
    assert rel(lam, lo) <= 1e-8, rel(lam, lo)
    for fa, fb in zip(op.fields(xs), o.fields(xo)):
        for fld, v in fb.items():
            if np.linalg.norm(v) > 0:
                assert rel(fa[fld], v) <= 1e-8, (name, fld, rel(fa[fld], v))
    op.close()


def test_direct_equals_krylov_to_its_tolerance():
    """The direct solve and the engine's own SQMR at a tightened tolerance agree
    (same operator, different solver): fields within 1e-9 on the 4x4 c4 layout."""
    kw = dict(SMALL["c4_params"], steps=2)
    a = pf.FetiOperator(**dict(kw, krylov="direct"))
    b = pf.FetiOperator(**dict(kw, tol=1e-13, max_iter=3000))
    for _ in range(2):
        a.step(), b.step()
        (xa, la), (xb, lb) = a.state(), b.state()
        assert rel(la, lb) <= 1e-9
        for u, v in zip(xa, xb):
            assert rel(u, v) <= 1e-9
    a.close(), b.close()


def test_direct_c2_full_size_all_steps():
    """BASELINE c2 at its own size (n_lambda 576), all 10 steps, against the
    oracle's FETI at tol 1e-13 (a live CPU run): fields and lambda within 1e-8."""
    import oracle_lib as ol
    kw = dict(pf.BASELINE_CONFIGS["c2"])
    op = pf.FetiOperator(**dict(kw, krylov="direct"))
    o = ol.Oracle(**dict(kw, tol=1e-13, max_iter=2000))
    o.run(kw["steps"])
    for k in range(1, kw["steps"] + 1):
        rep = op.step()
        assert rep["iterations"] == 0 and rep["true_residual"] <= 1e-11, (k, rep)
        xs, lam = op.state()
        xo, lo = o.state(k)
        assert rel(lam, lo) <= 1e-8, (k, rel(lam, lo))
        for u, v in zip(xs, xo):
            assert rel(u, v) <= 1e-8, k
    op.close()


@pytest.mark.parametrize("name", ["full_c3", "full_c5"])
def test_direct_full_size_matches_fixture(name):
    """c3 (nu = 0.49999) and c5 (log-normal permeability) at BASELINE size:
    the direct step against the oracle's SQMR fixture, at the fixture's bars
    (1e-8, or 10x the oracle's own measured tolerance sensitivity)."""
    from test_gpu_fullsize import FIELDS as FF, bar, global_fields, load as fload
    z, cfg = fload(name)
    op = pf.FetiOperator(**dict(cfg, krylov="direct"))
    for k in range(1, int(z["steps"]) + 1):
        rep = op.step()
        assert rep["iterations"] == 0 and rep["true_residual"] <= 1e-10, (k, rep)
        xs, lam = op.state()
        assert rel(lam, z[f"lambda{k}"]) <= bar(z, k, 4), (k, rel(lam, z[f"lambda{k}"]))
        g = global_fields(op, xs)
        for j, fld in enumerate(FF):
            b = bar(z, k, j)
            idx = z[f"idx_{fld}{k}"]
            assert rel(g[fld][idx], z[f"val_{fld}{k}"]) <= b, (k, fld)
    op.close()


def test_direct_pf_krylov_caller_rhs():
    """pf_krylov (feti_pcg's entry point) on a direct context: a caller rhs and
    lambda0 give lambda with P(rhs - F lambda) ~ 0 and G_c^T lambda = G_c^T lambda0 (= 0)."""
    kw = dict(SMALL["c4_params"], krylov="direct")
    op = pf.FetiOperator(**kw)
    rng = np.random.default_rng(7)
    rhs = rng.uniform(-1, 1, op.n_lambda)
    lam0 = np.zeros(op.n_lambda)
    lam, rep = op.krylov(rhs, lam0, 1e-10, 10)
    assert rep["iterations"] == 0
    r = op.project(rhs - op.apply(lam))
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(op.project(rhs))
    op.close()


def test_direct_rejects_large_and_sharded():
    """n_lambda above the dense cap (BASELINE c4: 162,378) is a ConfigError (PF_INVALID)."""
    with pytest.raises(pf.ConfigError):
        pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c4"], krylov="direct"))
