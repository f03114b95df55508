"""The oracle restatement pinned to the reference ITSELF (CPU).

tests/golden/ref_*.npz come from the unmodified reference headers
(/root/reference/proj/include/porofeti) compiled against the Eigen-API shim
(oracle/ref/, recipe oracle/ref/Makefile, generator oracle/ref/make_ref_golden.py):
the reference's own build_discretization, assembly, FetiOperator, feti_pcg,
StepSolver::advance and verify.hpp produced them.  Each fixture also stores
how far the reference moves when its LU uses another, equally valid
elimination order (spread_*): the rounding envelope of the reference's own
answer.  The oracle must sit inside 10x that envelope (floor 1e-10) on every
field of every stored step, and match the reference's iteration counts
(+-2 on BASELINE config 1; see ref_cases.ill_conditioned for the E=1e4 cases).
"""
import numpy as np
import pytest

import oracle_lib as ol
from ref_cases import CASES, FIELDS, ill_conditioned, iteration_window, load, named_fields, rel


def envelope(z, f, steps):
    return max(float(z[f"spread_{f}{k}"]) for k in range(1, steps + 1))


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_reference_run(name):
    kw = CASES[name]
    z = load(name)
    o = ol.Oracle(**kw)
    assert o.n_lambda == int(z["n_lambda"])
    # operator and preconditioner of the reference on its seeded multiplier
    cond_floor = 1e-9 if ill_conditioned(name) else 1e-12
    assert rel(o.apply(z["apply_in"]), z["apply_out"]) <= cond_floor
    assert rel(o.precond(z["apply_in"]), z["precond_out"]) <= cond_floor
    n = kw["steps"]
    o.run(n)
    for k in range(1, n + 1):
        xs, lam = o.state(k)
        f = o.fields(xs)
        got = named_fields(f[0], f[1], lam)
        for fld in FIELDS:
            ref = z[f"{fld}{k}"]
            if np.linalg.norm(ref) == 0:
                assert np.linalg.norm(got[fld]) == 0
                continue
            bar = max(1e-10, 10.0 * envelope(z, fld, n))
            assert rel(got[fld], ref) <= bar, (name, k, fld, rel(got[fld], ref), bar)
        it, it_ref = o.report(k)["iterations"], int(z[f"iters{k}"])
        if name == "c1_schur":
            assert abs(it - it_ref) <= 2, (k, it, it_ref)
        elif name == "c1_generalized":
            lo, hi = iteration_window(z[f"hist{k}"], 1e-10)
            assert lo <= it <= hi, (k, it, it_ref, lo, hi)
        else:
            assert 0.75 * it_ref <= it <= it_ref + 2, (k, it, it_ref)


def test_reference_feti_equals_its_monolithic_solve():
    """The reference's FETI path equals its own MonolithicSolver (SPEC AC1) on
    c1 -- a check of the fixtures -- and the oracle's monolithic restatement
    equals the reference's monolithic solve."""
    zf, zm = load("c1_schur"), load("c1_monolithic")
    for k in range(1, 6):
        for fld in FIELDS:
            if np.linalg.norm(zm[f"{fld}{k}"]) > 0:
                assert rel(zf[f"{fld}{k}"], zm[f"{fld}{k}"]) <= 1e-8, (k, fld)
    o = ol.Oracle(**CASES["c1_schur"])
    x, lam = o.monolithic_step()
    f = o.fields(x)
    got = named_fields(f[0], f[1], lam)
    for fld in FIELDS:
        if np.linalg.norm(zm[f"{fld}1"]) > 0:
            assert rel(got[fld], zm[f"{fld}1"]) <= 1e-10, fld


def test_paper_table3_anchor_settled_by_the_reference():
    """SPEC's accuracy anchor (||u - u_h|| ~ 3.4e-5 at h = 1/8,
    P2, nu = 0.2) against the reference's OWN mms scenario run to T = 1e-2:
    the reference gives L-inf(L2) 4.6e-3, the oracle the same number -- the
    gap to the paper is the reference's (its mms field sin 2 pi x sin 2 pi y
    is interpolated at h = 1/8), not the restatement's."""
    z = load("mms_m8")
    ref_linf = float(z["linf_err_u"])
    assert 4e-3 < ref_linf < 5e-3
    kw = dict(CASES["mms_m8"], steps=int(z["N"]))
    o = ol.Oracle(**kw)
    o.run(kw["steps"])
    linf = max(o.errors(k)[0] for k in range(1, kw["steps"] + 1))
    assert abs(linf - ref_linf) <= 1e-6 * ref_linf, (linf, ref_linf)
    assert linf > 10 * 3.4e-5  # the paper's number is not reproduced by the reference either
