"""CPU tests of the engine's host side and C ABI (no GPU needed).

* the shared library loads and exports every symbol include/porofeti_b200.h
  declares;
* the host discretisation (partition, numbering, constraints, mortar
  multipliers, saddle patterns) equals the oracle's on the BASELINE layouts;
* the symbolic analysis (nested dissection, supernodes, multi-level task
  schedule, slots, contribution/fold lists) solves exactly: the host emulation
  of the device schedule reproduces the oracle's subdomain solves;
* without a CUDA device the engine refuses to run (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

import oracle_lib as ol
import paper_2509_06673_b200 as pf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "porofeti_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|long long)\s+(pf_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = pf.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(pf.CudaUnavailableError):
        pf.FetiOperator(**pf.BASELINE_CONFIGS["c1"])


@pytest.mark.parametrize("name,kw", [
    ("c1", dict(pf.BASELINE_CONFIGS["c1"])),
    ("c2-small", dict(pf.BASELINE_CONFIGS["c2"], mesh_n=16)),
    ("c4-small", dict(pf.BASELINE_CONFIGS["c4"], mesh_n=32, SX=4, SY=4)),
    ("p1-multi", dict(pf.BASELINE_CONFIGS["c1"], mesh_n=24, SX=3, SY=4)),
    ("c5-small", dict(pf.BASELINE_CONFIGS["c5"], mesh_n=32, SX=4, SY=4)),
])
def test_host_discretisation_matches_oracle(name, kw):
    o = ol.Oracle(**kw)
    cfg = pf.make_config(**kw)
    for s in range(o.n_sub):
        d = pf.debug_disc(cfg, s)
        assert (d["n_lambda"], d["n_lambda_u"]) == (o.n_lambda, o.n_lambda_u)
        G = o.matrix(s, "G")
        gl, gc, gv = d["G"]
        Gp = sp.csr_matrix((gv, (gl, gc)), shape=G.shape)
        assert abs(G - Gp).max() <= 1e-15  # identical mortar rows and signs
        K = o.matrix(s, "K")
        n = K.shape[0]
        Kp = sp.csr_matrix((np.ones(len(d["K_col"])), d["K_col"], d["K_ptr"][:n + 1]), shape=K.shape)
        assert ((abs(K) > 0).astype(int) - (Kp > 0).astype(int)).max() <= 0  # pattern contains oracle's


@pytest.mark.parametrize("name,kw,subs", [
    ("c1", dict(pf.BASELINE_CONFIGS["c1"]), [0, 1]),
    ("c2-64", dict(pf.BASELINE_CONFIGS["c2"], mesh_n=32), [0, 3]),
    ("c4-sub", dict(pf.BASELINE_CONFIGS["c4"], mesh_n=64, SX=2, SY=2), [0, 2]),
])
@pytest.mark.parametrize("cap", [4096, 40000])
def test_task_schedule_emulation_solves(name, kw, subs, cap):
    o = ol.Oracle(**kw)
    cfg = pf.make_config(**kw)
    for s in subs:
        if o.subs[s]["floating"]:
            continue
        d = pf.debug_disc(cfg, s)
        K = o.matrix(s, "K")
        n = K.shape[0]
        ic = d["dof_ic"][:2 * n].reshape(-1, 2)
        b = np.random.default_rng(s).uniform(-1, 1, n)
        xo = o.local_solve(s, b)
        for mode in (0, 1):
            x, stats = pf.debug_factor_solve(K, ic, b, mode=mode, task_cap=cap)
            assert np.linalg.norm(K @ x - b) <= 1e-12 * np.linalg.norm(b)
            assert np.linalg.norm(x - xo) <= 1e-12 * np.linalg.norm(xo)
        assert stats[1] > 1  # a real task schedule


def test_mortar_gram_schedule_emulation():
    """The lambda-space Gram matrix sum_s G_s G_s^T (mortar scaling) through
    the same symbolic path (generic graph with cross-point cliques)."""
    kw = dict(pf.BASELINE_CONFIGS["c4"], mesh_n=64, SX=8, SY=8)
    o = ol.Oracle(**kw)
    cfg = pf.make_config(**kw)
    A = None
    for s in range(o.n_sub):
        G = o.matrix(s, "G")
        A = G @ G.T if A is None else A + G @ G.T
    A = A.tocsr()
    m, ifs = o.mults()
    # multiplier coordinates on the global half-cell grid from the interface table
    n_sub_x = kw["SX"]
    cx = kw["mesh_n"] // kw["SX"]
    ic = np.zeros((o.n_lambda, 2), np.int32)
    for i, (f, k, comp) in enumerate(m):
        a, b, horiz, pp = ifs[f]
        sx, sy = a % n_sub_x, a // n_sub_x
        gi = sx * cx + k if horiz else (sx + 1) * cx
        gj = (sy + 1) * cx if horiz else sy * cx + k
        ic[i] = (2 * gi, 2 * gj)
    b = np.random.default_rng(5).uniform(-1, 1, o.n_lambda)
    x, stats = pf.debug_factor_solve(A, ic, b, mode=1, task_cap=4096)
    assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b)
    assert stats[1] > 4


def test_baseline_config_table_matches_oracle_table():
    for name, kw in pf.BASELINE_CONFIGS.items():
        okw = ol.BASELINE_CONFIGS[name]
        for k, v in okw.items():
            assert kw[k] == v, (name, k)
