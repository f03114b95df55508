"""The wide per-step factor sweep (pf_sweep.cuh k_sweep_w: V same-type
subdomains per warp task, each factor value streamed once for V interleaved
right-hand sides) against the scalar batched sweep it replaces
(SubdomainFactorization::solve, feti.hpp:38, batched): every member's
arithmetic is the scalar kernel's operation for operation, so whole time steps
must agree BITWISE, for both widths, with floating subdomains (fixing dofs
zeroed), through the FETI Krylov path and the direct interface solve."""
import numpy as np
import pytest

import paper_2509_06673_b200 as pf

pytestmark = pytest.mark.gpu


def run(kw, env, monkeypatch, steps=2):
    for k in ("PF_NO_WIDE", "PF_WIDE"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    op = pf.FetiOperator(**kw)
    width = op.info.sweep_width
    out = []
    for _ in range(steps):
        rep = op.step()
        xs, lam = op.state()
        out.append((np.concatenate(xs), lam.copy(), rep["iterations"]))
    op.close()
    return width, out


@pytest.mark.parametrize("width", [2, 4])
@pytest.mark.parametrize("name,krylov", [("c4", "auto"), ("c3", "auto"), ("c4", "direct")])
def test_wide_sweep_bitwise_equals_scalar(name, krylov, width, monkeypatch):
    kw = dict(pf.BASELINE_CONFIGS[name], mesh_n=64, SX=8, SY=8, steps=2, krylov=krylov)
    w0, a = run(kw, {"PF_NO_WIDE": "1"}, monkeypatch)
    w1, b = run(kw, {"PF_WIDE": str(width)}, monkeypatch)
    assert w0 == 1 and w1 == width
    for (xa, la, ia), (xb, lb, ib) in zip(a, b):
        assert ia == ib
        assert np.array_equal(la, lb)
        assert np.array_equal(xa, xb)


@pytest.mark.parametrize("width", [2, 4])
def test_wide_sweep_per_level_check(width, monkeypatch):
    """pf_debug_wide_check: the wide and the scalar sweep on the current
    right-hand side differ in no entry of any elimination-tree level."""
    monkeypatch.delenv("PF_NO_WIDE", raising=False)
    monkeypatch.setenv("PF_WIDE", str(width))
    op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c3"], mesh_n=64, SX=8, SY=8, steps=2))
    op.step()
    lv = op.wide_check()
    assert lv.shape[0] >= 2 and np.all(lv == 0.0), lv
    op.close()


def test_wide_sweep_default_rule(monkeypatch):
    """The width rule: the largest of {4, 2} whose zero padding stays under
    30 % and that leaves at least three groups per SM (the sweep is bound by
    the dependency chain inside a task: fewer, wider tasks only pay while they
    still fill the machine).  BASELINE c4 (1024 subdomains) takes width 2;
    smaller partitions, one-member types and subdomains with their own factor
    values (c5: per-element permeability) keep the scalar sweep."""
    for k in ("PF_NO_WIDE", "PF_WIDE"):
        monkeypatch.delenv(k, raising=False)
    op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c4"], steps=1))
    assert op.info.sweep_width == 2 and op.info.sweep_wide_problems >= 512
    scalar = None
    t_wide = op.bench(8, 3, 10)[0]
    op.close()
    monkeypatch.setenv("PF_NO_WIDE", "1")
    op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS["c4"], steps=1))
    t_scalar = op.bench(8, 3, 10)[0]
    op.close()
    monkeypatch.delenv("PF_NO_WIDE")
    print(f"c4 per-step sweep: scalar {t_scalar:.3f} ms, wide (2) {t_wide:.3f} ms")
    assert t_wide < 1.05 * t_scalar  # measured 2.7 vs 3.4 ms
    for kw in (dict(pf.BASELINE_CONFIGS["c4"], mesh_n=128, SX=16, SY=16, steps=1),   # 256 subdomains: too few groups
               dict(pf.BASELINE_CONFIGS["c2"], mesh_n=32, steps=1),                  # 2x2: four one-member types
               dict(pf.BASELINE_CONFIGS["c5"], mesh_n=64, SX=8, SY=8, steps=1)):     # own factor values
        op = pf.FetiOperator(**kw)
        assert op.info.sweep_width == 1
        op.close()
