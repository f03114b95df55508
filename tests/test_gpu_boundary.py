"""The drop-in boundary beyond pf_step: the reference's per-step pieces one by
one (interface_rhs -> feti_pcg -> back_substitute, timeloop.hpp:163-176), the
residual history, set_precond, the field-named snapshot, caller-supplied
loads, the element-level entry point, and the C++ shim compiled and linked
against the library -- checked against the reference's own outputs
(tests/golden/ref_*.npz, the unmodified reference headers over the Eigen-API
shim) and the oracle."""
import os
import subprocess

import numpy as np
import pytest

import paper_2509_06673_b200 as pf
from ref_cases import CASES, FIELDS, load, rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_step_pieces_match_reference_step():
    """interface_rhs, feti_pcg, back_substitute called one by one equal the
    device step and the reference's own first step of c1 (feti-schur)."""
    z = load("c1_schur")
    kw = CASES["c1_schur"]
    a = pf.FetiOperator(**kw)
    ra = a.step()
    xa, la = a.state()
    b = pf.FetiOperator(**kw)
    F = b.interface_rhs()
    lam, rep = pf.feti_pcg(b, F, np.zeros(b.n_lambda), 1e-10, 500)
    x = b.back_substitute(lam)
    assert rep["iterations"] == ra["iterations"]
    assert rel(lam, la) <= 1e-13 and rel(x, np.concatenate(xa)) <= 1e-13
    # the reference's residual history: same initial sqrt(r.z), same early decay
    h, hr = rep["residual_history"], z["hist1"]
    assert len(h) == rep["iterations"] + 1
    assert abs(h[0] - hr[0]) <= 1e-12 * hr[0]
    assert np.allclose(h[:10] / h[0], hr[:10] / hr[0], rtol=1e-6, atol=0)
    assert abs(rep["iterations"] - int(z["iters1"])) <= 2
    assert rel(lam, z["lambda1"]) <= 1e-8
    # back_substitute leaves the device state alone
    assert rel(b.state()[1], np.zeros(b.n_lambda)) == 0.0


def test_krylov_errors_like_reference():
    op = pf.FetiOperator(**CASES["c1_schur"])
    F = op.interface_rhs()
    with pytest.raises(pf.SolverError):  # tolerance must be positive (feti.hpp:265)
        op.krylov(F, np.zeros(op.n_lambda), 0.0, 10)
    with pytest.raises(pf.SolverError):  # not converged within max_iter
        op.krylov(F, np.zeros(op.n_lambda), 1e-10, 3)
    lam, rep = op.krylov(F, np.zeros(op.n_lambda), 1e-6, 500)  # another tolerance: graph re-captured
    assert rep["converged"] and rep["rel_residual"] <= 1e-6
    with pytest.raises(pf.ConfigError):
        op.krylov(F[:-1], np.zeros(op.n_lambda), 1e-10, 10)


def test_set_precond_matches_reference_preconditioners():
    zs, zg = load("c1_schur"), load("c1_generalized")
    op = pf.FetiOperator(**CASES["c1_schur"])
    x = zs["apply_in"]
    assert rel(op.apply_preconditioner(x), zs["precond_out"]) <= 1e-11
    op.set_precond("generalized")
    assert rel(op.apply_preconditioner(x), zg["precond_out"]) <= 1e-11
    op.set_precond("identity")
    assert np.array_equal(op.apply_preconditioner(x), x)
    op.set_precond("generalized")
    rep = op.step()
    _, lam = op.state()
    assert rel(lam, zg["lambda1"]) <= 1e-8 and rep["converged"]
    op.set_precond("dirichlet")
    assert rel(op.apply_preconditioner(x), zs["precond_out"]) <= 1e-11
    # the explicit local operators carry the Dirichlet blocks Sd_s whatever the
    # preconditioner at creation: a generalized context can switch to feti-schur's
    g = pf.FetiOperator(**CASES["c1_generalized"])
    g.set_precond("dirichlet")
    assert rel(g.apply_preconditioner(x), zs["precond_out"]) <= 1e-11
    # the implicit (factor-sweep) path builds the interior factors only for a
    # Dirichlet context: switching to it is refused, not undefined (REF: UB)
    os.environ["PF_FAPPLY"] = "implicit"
    try:
        h = pf.FetiOperator(**CASES["c1_generalized"])
        with pytest.raises(pf.ConfigError):
            h.set_precond("dirichlet")
        h.close()
    finally:
        del os.environ["PF_FAPPLY"]


def test_unpack_state_reference_names():
    z = load("c1_schur")
    op = pf.FetiOperator(**CASES["c1_schur"])
    op.step()
    snap = pf.unpack_state(op)
    assert snap["step"] == 1
    for fld in FIELDS:
        assert snap[fld].shape == z[f"{fld}1"].shape
        if np.linalg.norm(z[f"{fld}1"]) > 0:
            assert rel(snap[fld], z[f"{fld}1"]) <= 1e-8, fld
    assert np.array_equal(op.field("p", 0), snap["p"])
    with pytest.raises(pf.ConfigError):
        op.field("eta", 1)  # the elastic subdomain has no eta


def test_caller_loads_roundtrip_and_linearity():
    kw = dict(pf.BASELINE_CONFIGS["c4"], mesh_n=128, SX=4, SY=4, steps=2)
    a = pf.FetiOperator(**kw)
    a.step()
    xa, la = a.state()
    b = pf.FetiOperator(**kw)
    t1 = kw["dt"]
    F, Z, g = b.scenario_loads(t1)
    nF, nZ, nG = b.load_sizes()
    assert F.size == nF and Z.size == nZ and g.size == nG and np.abs(F).max() > 0
    b.set_loads(F, Z, g)
    b.step()
    xb, lb = b.state()
    assert np.array_equal(lb, la) and all(np.array_equal(u, v) for u, v in zip(xa, xb))
    # zero initial state: the step is linear in the loads
    c = pf.FetiOperator(**kw)
    c.set_loads(2.0 * F, 2.0 * Z, 2.0 * g)
    c.step()
    xc, lc = c.state()
    assert rel(lc, 2.0 * la) <= 1e-8
    assert rel(np.concatenate(xc), 2.0 * np.concatenate(xa)) <= 1e-8
    # constraint metadata: coordinates on the outer boundary, components in {-1, 0, 1}
    idx, comp, xy = c.constraints(0)
    assert idx.size and set(np.unique(comp)) <= {-1, 0, 1}
    assert np.all((np.isclose(xy, 0.0) | np.isclose(xy, 1.0)).any(axis=1))


def test_local_matrices_on_device_match_oracle_and_reference_kats():
    """The element-level entry point (elements.hpp:152-230) on the device:
    against the oracle's restatement on random triangles, and the reference's
    own known answers (tests/test_elements.cpp:144-230): the P1 mass matrix
    A/12 [[2,1,1],[1,2,1],[1,1,2]], exactly three rigid modes in the elastic
    kernel, zero row sums of the diffusion matrix."""
    import oracle_lib as ol
    rng = np.random.default_rng(7)
    for order in (1, 2):
        for _ in range(4):
            tri = rng.uniform(-1, 1, 6)
            if abs((tri[2] - tri[0]) * (tri[5] - tri[1]) - (tri[4] - tri[0]) * (tri[3] - tri[1])) < 0.1:
                continue
            d = pf.local_matrices(tri, 0.77, order, kperm=1.3, mu_f=0.9)
            t3 = tri.reshape(3, 2)
            assert rel(d["elastic"], ol.local_elastic(t3, 0.77, order)) <= 1e-13
            assert rel(d["div"], ol.local_div(t3, order)) <= 1e-13
            assert rel(d["mass"], ol.local_mass(t3)) <= 1e-13
            assert rel(d["diffusion"], ol.local_diffusion(t3, 1.3 * np.eye(2), 0.9)) <= 1e-13
            area = 0.5 * abs((tri[2] - tri[0]) * (tri[5] - tri[1]) - (tri[4] - tri[0]) * (tri[3] - tri[1]))
            assert np.allclose(d["mass"], area / 12 * (np.ones((3, 3)) + np.eye(3)), rtol=0, atol=1e-12 * area)
            ev = np.linalg.eigvalsh(0.5 * (d["elastic"] + d["elastic"].T))
            assert np.sum(np.abs(ev) < 1e-10 * np.abs(ev).max()) == 3
            assert np.abs(d["diffusion"].sum(axis=1)).max() <= 1e-13 * np.abs(d["diffusion"]).max()
    with pytest.raises(pf.ConfigError):
        pf.local_matrices([0, 0, 1, 1, 2, 2], 1.0, 1)


def test_cpp_shim_example_builds_and_matches_reference(tmp_path):
    """examples/run_c1.cpp (the header-only C++ shim over the C ABI) compiled
    and linked here; its output equals the reference's own c1 run."""
    exe = tmp_path / "run_c1"
    lib = os.path.join(ROOT, "paper_2509_06673_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "run_c1.cpp"), "-L" + lib, "-lporofeti_b200",
                    "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=300).stdout
    z = load("c1_schur")
    lines = out.strip().splitlines()
    pieces = lines[0].split()
    assert pieces[0] == "pieces" and abs(int(pieces[4]) - int(z["iters1"])) <= 2
    assert abs(float(pieces[10]) - np.linalg.norm(z["lambda1"])) <= 1e-8 * np.linalg.norm(z["lambda1"])
    steps = [ln.split() for ln in lines[1:] if ln.startswith("step ")]
    assert len(steps) == 5
    # SolverChoice::monolithic through the shim: the reference's own monolithic
    # run's error norms (tests/golden/ref_c1_monolithic.npz), no iterations
    zm = load("c1_monolithic")
    mono = [ln.split() for ln in lines[1:] if ln.startswith("monolithic ")]
    assert len(mono) == 5
    for k, f in enumerate(mono, start=1):
        assert int(f[1]) == k and int(f[3]) == 0 and float(f[5]) <= 1e-12
        assert abs(float(f[7]) - float(zm[f"err_u{k}"])) <= 1e-8 * float(zm[f"err_u{k}"])
        assert abs(float(f[9]) - float(zm[f"err_p{k}"])) <= 1e-8 * float(zm[f"err_p{k}"])
    for k, f in enumerate(steps, start=1):
        assert int(f[1]) == k and abs(int(f[3]) - int(z[f"iters{k}"])) <= 2
        assert float(f[7]) <= 1e-10  # true residual
        assert abs(float(f[9]) - float(z[f"err_u{k}"])) <= 1e-6 * float(z[f"err_u{k}"])
        assert abs(float(f[11]) - float(z[f"err_p{k}"])) <= 1e-6 * float(z[f"err_p{k}"])
