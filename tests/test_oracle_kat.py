"""Pins the CPU oracle to the reference's own known-answer tests.

Every test here re-expresses one GTest of /root/reference/proj/tests
(test_elements.cpp:46-264, test_mesh.cpp:28-211) against the oracle's C++
restatement.  The element/mesh layer is the only part of the hot path that the
reference tests; the FETI layer is pinned by SPEC invariants in
test_oracle_feti.py.
"""
import math

import numpy as np
import pytest

import oracle_lib as ol


def monomial_integral(a, b):  # test_elements.cpp:15-23
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


def random_triangle(rng):  # test_elements.cpp:25-35 (|2 area| > 0.2)
    while True:
        t = rng.uniform(-1.0, 1.0, size=(3, 2))
        a2 = (t[1, 0] - t[0, 0]) * (t[2, 1] - t[0, 1]) - (t[2, 0] - t[0, 0]) * (t[1, 1] - t[0, 1])
        if abs(a2) > 0.2:
            return t


def random_reference_point(rng):
    while True:
        p = rng.uniform(0.0, 1.0, size=2)
        if p.sum() <= 1.0:
            return p


# ------------------------------------------------------------------ basis --
def test_basis_lagrange_property():  # test_elements.cpp:46-61
    v, _ = ol.eval_basis(1, 0.0, 0.0)
    assert v.tolist() == [1.0, 0.0, 0.0]
    nodes = [(0, 0), (1, 0), (0, 1), (0.5, 0), (0.5, 0.5), (0, 0.5)]
    for n, (x, y) in enumerate(nodes):
        v, _ = ol.eval_basis(2, x, y)
        for i in range(6):
            assert abs(v[i] - (1.0 if i == n else 0.0)) < 1e-14


def test_basis_partition_of_unity_and_gradient_sum():  # test_elements.cpp:63-82
    rng = np.random.default_rng(7)
    for order in (1, 2):
        for _ in range(100):
            p = random_reference_point(rng)
            v, g = ol.eval_basis(order, *p)
            assert abs(v.sum() - 1.0) < 1e-13
            assert np.linalg.norm(g.sum(axis=0)) < 1e-13


def test_basis_outside_point_rejected():  # test_elements.cpp:84-89
    with pytest.raises(ol.OracleError):
        ol.eval_basis(1, 0.7, 0.7)
    with pytest.raises(ol.OracleError):
        ol.eval_basis(3, 0.1, 0.1)


# ------------------------------------------------------------- quadrature --
def test_quadrature_low_order_rules():  # test_elements.cpp:91-110
    p, w = ol.triangle_rule(1)
    assert len(w) == 1 and abs(p[0, 0] - 1 / 3) < 1e-15 and w[0] == 0.5
    p, w = ol.triangle_rule(2)
    assert len(w) == 3 and all(x == 1 / 6 for x in w)
    assert abs((w * p[:, 0]).sum() - monomial_integral(1, 0)) < 1e-15
    assert abs((w * p[:, 1]).sum() - monomial_integral(0, 1)) < 1e-15
    assert abs((w * p[:, 0] ** 2).sum() - monomial_integral(2, 0)) < 1e-15


def test_quadrature_monomial_exactness():  # test_elements.cpp:112-130
    for degree in range(1, 5):
        p, w = ol.triangle_rule(degree)
        assert abs(w.sum() - 0.5) < 1e-14
        for a in range(degree + 1):
            for b in range(degree + 1 - a):
                acc = (w * p[:, 0] ** a * p[:, 1] ** b).sum()
                assert abs(acc - monomial_integral(a, b)) < 1e-13, (degree, a, b)
    with pytest.raises(ol.OracleError):
        ol.triangle_rule(5)


def test_quadrature_edge_rules():  # test_elements.cpp:132-142
    for degree in (1, 2, 3, 4, 5):
        p, w = ol.edge_rule(degree)
        for k in range(degree + 1):
            assert abs((w * p ** k).sum() - 1.0 / (k + 1)) < 1e-14


# ---------------------------------------------------------- local matrices --
def test_local_mass_analytic():  # test_elements.cpp:144-159
    rng = np.random.default_rng(21)
    for _ in range(10):
        t = random_triangle(rng)
        a2 = (t[1, 0] - t[0, 0]) * (t[2, 1] - t[0, 1]) - (t[2, 0] - t[0, 0]) * (t[1, 1] - t[0, 1])
        area = 0.5 * abs(a2)
        m = ol.local_mass(t)
        expect = np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]]) * area / 12.0
        assert np.abs(m - expect).max() < 1e-12 * area
        assert (m >= 0).all()


def test_local_div_on_constant_field():  # test_elements.cpp:161-174
    rng = np.random.default_rng(22)
    for order in (1, 2):
        t = random_triangle(rng)
        b = ol.local_div(t, order)
        nb = 3 if order == 1 else 6
        c = np.tile([0.7, -1.3], nb)
        assert np.linalg.norm(b @ c) < 1e-12


def test_local_elastic_kernel_is_rigid_modes():  # test_elements.cpp:176-216
    rng = np.random.default_rng(23)
    for order in (1, 2):
        for _ in range(5):
            t = random_triangle(rng)
            a = ol.local_elastic(t, 123.0, order)
            assert np.abs(a - a.T).max() < 1e-14 * np.abs(a).max()
            ev = np.linalg.eigvalsh(a)
            scale = np.abs(ev).max()
            assert (np.abs(ev) < 1e-10 * scale).sum() == 3
            assert ev.min() > -1e-10 * scale
            nodes = list(t)
            if order == 2:
                nodes += [0.5 * (t[0] + t[1]), 0.5 * (t[1] + t[2]), 0.5 * (t[2] + t[0])]
            rot = np.array([[-n[1], n[0]] for n in nodes]).reshape(-1)
            tx = np.tile([1.0, 0.0], len(nodes))
            ty = np.tile([0.0, 1.0], len(nodes))
            for v in (rot, tx, ty):
                assert np.linalg.norm(a @ v) < 1e-10 * scale


def test_local_diffusion_row_sums_and_symmetry():  # test_elements.cpp:218-230
    rng = np.random.default_rng(24)
    K = [[2.0, 0.3], [0.3, 1.5]]
    for _ in range(5):
        t = random_triangle(rng)
        f = ol.local_diffusion(t, K, 0.7)
        assert np.abs(f - f.T).max() < 1e-13 * np.abs(f).max()
        assert np.abs(f.sum(axis=1)).max() < 1e-13 * np.abs(f).max()


def test_local_degenerate_triangle_rejected():  # test_elements.cpp:232-235
    with pytest.raises(ol.OracleError) as e:
        ol.local_mass([[0, 0], [1, 1], [2, 2]])
    assert e.value.code == 4  # AssemblyError


def test_local_interface_p1_analytic():  # test_elements.cpp:237-246
    m = ol.local_interface((0.25, 0.5), (0.75, 0.5), 1)
    expect = np.array([[2, 1], [1, 2]]) * 0.5 / 6.0
    assert np.abs(m - expect).max() < 1e-14
    assert abs(m.sum() - 0.5) < 1e-14


def test_local_interface_p2_analytic():  # test_elements.cpp:248-257
    L = 0.375
    m = ol.local_interface((0.0, 0.5), (L, 0.5), 2)
    expect = np.array([[1 / 6, 0, 1 / 3], [0, 1 / 6, 1 / 3]]) * L
    assert np.abs(m - expect).max() < 1e-14


def test_local_interface_scales_linearly():  # test_elements.cpp:259-264
    small = ol.local_interface((0, 0), (0.25, 0), 1)
    big = ol.local_interface((0, 0), (0.75, 0), 1)
    assert np.abs(3 * small - big).max() < 1e-14
    with pytest.raises(ol.OracleError):
        ol.local_interface((0, 0), (0, 0), 1)


# ------------------------------------------------------------------- mesh --
def test_mesh_structured_grid_counts():  # test_mesh.cpp:28-33
    m = ol.Mesh(0, (0, 0, 1, 0.5), 8, 4)
    assert m.counts() == (45, 64, 8 * 5 + 9 * 4 + 32)


def test_mesh_smallest_grid():  # test_mesh.cpp:35-39
    m = ol.Mesh(1, (0, 0, 1, 1), 1, 1)
    assert m.counts()[:2] == (4, 2)


def test_mesh_positive_areas_and_partition():  # test_mesh.cpp:41-48
    for n in (1, 2, 5, 8, 13):
        rect = (-0.5, 0.25, 2.0, 1.0)
        m = ol.Mesh(0, rect, n, n + 1)
        _, a = m.triangles()
        assert (a > 0).all()
        area = (rect[2] - rect[0]) * (rect[3] - rect[1])
        assert abs(a.sum() - area) < 1e-12 * area


def test_mesh_rejects_bad_input():  # test_mesh.cpp:50-54
    for args in (((0, 0, 1, 1), 0, 4), ((0, 0, 1, 1), 4, -1), ((0, 0, 0, 1), 4, 4)):
        with pytest.raises(ol.OracleError) as e:
            ol.Mesh(0, *args)
        assert e.value.code == 4


def test_mesh_refinement_nesting():  # test_mesh.cpp:56-68
    c = ol.Mesh(0, (0, 0, 1, 0.5), 6, 3).vertices()
    f = ol.Mesh(0, (0, 0, 1, 0.5), 12, 6).vertices()
    for v in c:
        assert np.abs(f - v).max(axis=1).min() < 1e-12


def test_mesh_boundary_tagging():  # test_mesh.cpp:70-81
    m = ol.Mesh(0, (0, 0, 1, 0.5), 8, 4)
    m.tag(0, 0.5)
    e, mask, pt, iface, mid = m.boundary()
    assert len(e) == 2 * 8 + 2 * 4
    assert iface.sum() == 8


def test_mesh_barry_mercer_layout_tags():  # test_mesh.cpp:83-100
    m = ol.Mesh(0, (0, 0, 1, 0.5), 8, 4)
    m.tag(1)
    e, mask, pt, iface, mid = m.boundary()
    for k in range(len(e)):
        if abs(mid[k, 1] - 0.5) < 1e-9:
            assert iface[k]
        elif abs(mid[k, 1]) < 1e-9:
            assert mask[k] == 2 and pt[k] == 1
        else:
            assert mask[k] == 1 and pt[k] == 1


def test_mesh_untaggable_edge_throws():  # test_mesh.cpp:102-108
    m = ol.Mesh(0, (0, 0, 1, 0.5), 2, 1)
    with pytest.raises(ol.OracleError) as e:
        m.tag(3)
    assert e.value.code == 4


def test_dofmap_counts_and_orders():  # test_mesh.cpp:110-122
    m = ol.Mesh(0, (0, 0, 1, 0.5), 8, 4)
    ne = m.counts()[2]
    nn, nd, _ = m.dofmap(0, 2)
    assert nn == 45 + ne and nd == 2 * (45 + 108)
    tiny = ol.Mesh(0, (0, 0, 1, 1), 1, 1)
    assert tiny.dofmap(3, 1)[1] == 4
    with pytest.raises(ol.OracleError):
        m.dofmap(0, 3)
    with pytest.raises(ol.OracleError):
        m.dofmap(3, 2)


def test_dofmap_per_subdomain_field_lists():  # test_mesh.cpp:124-129
    # P carries u, xi, eta, p; E carries u, xi: P saddle dim = n_u + 3 n_s, E = n_u + n_s
    o = ol.Oracle(mesh_n=8, SX=1, SY=2, order=2, steps=1)
    P, E = o.subs
    assert P["dim"] == P["n_u"] + 3 * P["n_s"] and E["dim"] == E["n_u"] + E["n_s"]


def _tagged_pair(nxp, nxe):
    P = ol.Mesh(0, (0, 0, 1, 0.5), nxp, max(1, nxp // 2))
    E = ol.Mesh(1, (0, 0.5, 1, 1), nxe, max(1, nxe // 2))
    P.tag(0, 0.5)
    E.tag(0, 0.5)
    return P, E


def test_interface_pairing_conforming_counts():  # test_mesh.cpp:143-158
    P, E = _tagged_pair(8, 8)
    pairs, nmult, ned = ol.pair(P, E, 1)
    assert len(pairs) == 9 and nmult == 9 and ned == 8
    pairs2, _, _ = ol.pair(P, E, 2)
    assert len(pairs2) == 17


def test_interface_pairing_nonconforming_rejected():  # test_mesh.cpp:160-165
    P, E = _tagged_pair(8, 16)
    with pytest.raises(ol.OracleError) as e:
        ol.pair(P, E, 1)
    assert e.value.code == 4


def test_interface_pairing_swap_symmetry():  # test_mesh.cpp:167-178
    P, E = _tagged_pair(4, 4)
    ab, _, _ = ol.pair(P, E, 2)
    ba, _, _ = ol.pair(E, P, 2)
    assert (ab[:, 0] == ba[:, 1]).all() and (ab[:, 1] == ba[:, 0]).all()


def test_interface_pairing_missing_interface_fails_loudly():  # test_mesh.cpp:180-191
    P = ol.Mesh(0, (0, 0, 1, 0.5), 4, 2)
    E = ol.Mesh(1, (0, 0.5, 1, 1), 4, 2)
    P.tag(4)
    E.tag(4)
    with pytest.raises(ol.OracleError):
        ol.pair(P, E, 1)


def test_interface_pairing_masks_match():  # test_mesh.cpp:193-211
    P, E = _tagged_pair(6, 6)
    pairs, _, _ = ol.pair(P, E, 2)
    _, _, onP = P.dofmap(0, 2)
    _, _, onE = E.dofmap(0, 2)
    assert onP[pairs[:, 0]].all() and onE[pairs[:, 1]].all()
    assert len(set(pairs[:, 0])) == len(pairs) == len(set(pairs[:, 1]))
    assert onP.sum() == len(pairs)
