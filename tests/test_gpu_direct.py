"""The direct interface solve (krylov="direct"): the GPU analogue of the
reference's monolithic solver (SolverChoice::monolithic, feti.hpp:313-440,
timeloop.hpp:139-160).

The coupled system is condensed exactly onto the multipliers.  Two variants
(the engine picks by size; PF_DIRECT=dense|sparse overrides, used here to run
both on the same layouts):
  * dense  (n_lambda <= 4096): F assembled dense from the explicit local
    operators and inverted once (signed Cholesky on the FP64 tensor cores;
    bordered by the rigid-mode constraint of the floating subdomains); every
    step is one GEMV;
  * sparse (BASELINE c3, c4, c5): a multifrontal block LDL^T over a nested
    dissection of the subdomain grid (pf_iface.hpp), fronts condensed on the
    FP64 tensor cores, one GEMV launch per tree depth and direction per step.
Both are followed by the same back-substitution as the FETI path.  Checked
against
  * the reference's OWN monolithic run of BASELINE config 1 (all 5 steps);
  * the oracle's monolithic restatement (dense LU of the whole coupled system)
    on multi-subdomain layouts with floating subdomains, pressure multipliers,
    nu = 0.49999 and the heterogeneous injection permeability;
  * the oracle's FETI solution at a tight Krylov tolerance at BASELINE c2's
    full size, and the full-size c3 / c4 / c5 fixtures (sparse variant).
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


VARIANTS = ("dense", "sparse")


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", list(SMALL))
def test_direct_matches_oracle_monolithic(name, variant, monkeypatch):
    """Step 1 vs the oracle's dense LU of the whole coupled system
    [blockdiag(K_s) G^T; G 0] (o_feti.hpp monolithic_solve): u, xi, eta, p and
    lambda within 1e-8 relative L2 per subdomain field."""
    import oracle_lib as ol
    monkeypatch.setenv("PF_DIRECT", variant)
    kw = dict(SMALL[name], krylov="direct")
    op = pf.FetiOperator(**kw)
    assert op.info.direct_sparse == (variant == "sparse")
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


@pytest.mark.parametrize("variant", VARIANTS)
def test_direct_equals_krylov_to_its_tolerance(variant, monkeypatch):
    """The direct solve and the engine's own SQMR at a tightened tolerance agree
    (same operator, different solver): fields within 1e-9 on the 4x4 c4 layout."""
    monkeypatch.setenv("PF_DIRECT", variant)
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


def test_sparse_equals_dense_on_ragged_partitions(monkeypatch):
    """The two variants on partitions that are not powers of two (3x2, 5x4:
    unbalanced interface trees, leaves at different depths) and without
    floating subdomains (3x2): lambda and every field within 1e-10."""
    for mesh, sx, sy in ((24, 3, 2), (40, 5, 4)):
        kw = dict(pf.BASELINE_CONFIGS["c4"], mesh_n=mesh, SX=sx, SY=sy, steps=2, krylov="direct")
        monkeypatch.setenv("PF_DIRECT", "dense")
        a = pf.FetiOperator(**kw)
        monkeypatch.setenv("PF_DIRECT", "sparse")
        b = pf.FetiOperator(**kw)
        assert b.info.direct_sparse == 1 and b.info.direct_fronts == sx * sy - 1
        for _ in range(2):
            ra, rb = a.step(), b.step()
            assert rb["true_residual"] <= 1e-11, rb
            (xa, la), (xb, lb) = a.state(), b.state()
            assert rel(lb, la) <= 1e-10
            for u, v in zip(xb, xa):
                assert rel(u, v) <= 1e-10
        a.close(), b.close()


@pytest.mark.parametrize("name", ["full_c3", "full_c5", "full_c4_m128", "full_c4"])
def test_direct_full_size_matches_fixture(name):
    """c3 (nu = 0.49999), c5 (log-normal permeability) and c4 (1024
    subdomains, 162,378 multipliers; also at mesh 128 with its true 32x32-cell
    subdomains) at BASELINE size: the direct step against the oracle's SQMR
    fixture, at the fixture's bars (1e-8, or 10x the oracle's own measured
    tolerance sensitivity).  The full-size configs take the sparse variant."""
    from test_gpu_fullsize import FIELDS as FF, bar, global_fields, load as fload
    z, cfg = fload(name)
    op = pf.FetiOperator(**dict(cfg, krylov="direct"))
    assert op.info.direct_sparse == (op.n_lambda > 4096)
    for k in range(1, int(z["steps"]) + 1):
        rep = op.step()
        assert rep["iterations"] == 0 and rep["true_residual"] <= 1e-10, (k, rep)
        xs, lam = op.state()
        assert rel(lam, z[f"lambda{k}"]) <= bar(z, k, 4), (k, rel(lam, z[f"lambda{k}"]))
        g = global_fields(op, xs)
        for j, fld in enumerate(FF):
            b = bar(z, k, j)
            if f"x{k}" in z.files:  # whole state in the fixture
                ref = op.fields(np.split(z[f"x{k}"], np.cumsum(z["dims"])[:-1]))
                r = np.concatenate([fi[fld] for fi in ref if fld in fi])
                assert rel(g[fld], r) <= b, (k, fld)
            else:
                idx = z[f"idx_{fld}{k}"]
                assert rel(g[fld][idx], z[f"val_{fld}{k}"]) <= b, (k, fld)
    op.close()


@pytest.mark.parametrize("variant", VARIANTS)
def test_direct_pf_krylov_caller_rhs(variant, monkeypatch):
    """pf_krylov (feti_pcg's entry point) on a direct context: a caller rhs and
    lambda0 give lambda with P(rhs - F lambda) ~ 0 and G_c^T lambda = G_c^T lambda0 (= 0)."""
    monkeypatch.setenv("PF_DIRECT", variant)
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


def test_dense_variant_rejects_large(monkeypatch):
    """The dense variant above its cap (BASELINE c4: 162,378 multipliers would
    need 211 GB) is a ConfigError (PF_INVALID); the size rule picks the sparse
    variant there."""
    monkeypatch.setenv("PF_DIRECT", "dense")
    with pytest.raises(pf.ConfigError):
        pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c4"], krylov="direct"))


def test_direct_c4_all_steps():
    """BASELINE c4, all 10 steps through the sparse direct interface solve:
    every step's true residual ||P(rhs - F lambda)|| / ||P rhs|| <= 1e-11 and
    the manufactured solution's error stays on the discretisation level."""
    op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c4"], krylov="direct"))
    assert op.info.direct_sparse == 1 and op.info.direct_fronts == 1023
    reps = pf.run_simulation(op)
    assert len(reps) == op.info.N
    assert all(r["iterations"] == 0 and r["true_residual"] <= 1e-11 for r in reps), reps
    eu, ep = op.errors()
    assert eu <= 1e-3 * op.info.T and ep <= 1e-3 * op.info.T, (eu, ep)
    op.close()
