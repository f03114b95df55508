"""CPU check of the algebra behind the engine's edge-local mortar Gram solve
(Engine::setup_qlocal, k_qlocal_y / k_qlocal_x), on the oracle's own G
matrices (BASELINE c4's subdomain size: 4x4 subdomains of 32x32 P2 cells):

  * W = sum_s G_s G_s^T is block diagonal over (interface, component) blocks
    -- banded, well conditioned -- plus couplings between END multipliers of
    different blocks only;
  * the far-corner entry of each block inverse is negligible (<= 1e-9 of the
    diagonal; 1e-13 here), so the Woodbury capacitance matrix is block diagonal
    over the cross-point groups;
  * W^-1 b = D^-1 b - D^-1 U K U^T D^-1 b with K = E (I + S E)^-1 per group
    reproduces a sparse direct solve to rounding.

This is the numpy restatement of what the device kernels apply; the GPU tests
(tests/test_gpu_qlocal.py) compare the kernels with the generic sparse factor.
"""
import numpy as np
import pytest

import oracle_lib as ol


def build_w(o):
    import scipy.sparse as sp
    n = o.n_lambda
    W = sp.csr_matrix((n, n))
    for s in range(len(o.subs)):
        G = o.matrix(s, "G")
        W = W + G @ G.T
    return W.tocsr()


def edge_local(W, mults):
    n = W.shape[0]
    key = mults[:, 0] * 4 + (mults[:, 2] + 1)
    blocks = {}
    for g in range(n):
        blocks.setdefault(int(key[g]), []).append(g)
    B = list(blocks.values())
    blk_of, pos_of = np.zeros(n, int), np.zeros(n, int)
    for e, idx in enumerate(B):
        for p, g in enumerate(idx):
            blk_of[g], pos_of[g] = e, p
    inv, conds, bands = [], [], []
    for idx in B:
        De = W[idx][:, idx].toarray()
        Di = np.linalg.inv(De)
        inv.append((Di + Di.T) / 2)
        conds.append(np.linalg.cond(De))
        nz = np.nonzero(De)
        bands.append(int(np.max(np.abs(nz[0] - nz[1]))))
    C = W.tocoo()
    off = [(r, c) for r, c, v in zip(C.row, C.col, C.data) if blk_of[r] != blk_of[c] and v != 0.0]
    ends = sorted({r for r, _ in off})
    par = {u: u for u in ends}

    def find(u):
        while par[u] != u:
            par[u] = par[par[u]]
            u = par[u]
        return u

    for r, c in off:
        par[find(r)] = find(c)
    groups = {}
    for u in ends:
        groups.setdefault(find(u), []).append(u)
    K = {}
    for root, mem in groups.items():
        k = len(mem)
        E, S = np.zeros((k, k)), np.zeros((k, k))
        for a, u in enumerate(mem):
            for b, v in enumerate(mem):
                if blk_of[u] != blk_of[v]:
                    E[a, b] = W[u, v]
                else:
                    S[a, b] = inv[blk_of[u]][pos_of[u], pos_of[v]]
        Kg = E @ np.linalg.inv(np.eye(k) + S @ E)
        K[root] = (mem, (Kg + Kg.T) / 2)
    drop = 0.0
    for e, idx in enumerate(B):
        en = [g for g in idx if g in par]
        for u in en:
            for v in en:
                if u < v and find(u) != find(v):
                    Di = inv[e]
                    drop = max(drop, abs(Di[pos_of[u], pos_of[v]]) / np.sqrt(Di[pos_of[u], pos_of[u]] * Di[pos_of[v], pos_of[v]]))

    def apply(b):
        y = np.zeros(n)
        for e, idx in enumerate(B):
            y[idx] = inv[e] @ b[idx]
        x = y.copy()
        for mem, Kg in K.values():
            t = Kg @ y[mem]
            for a, u in enumerate(mem):
                e = blk_of[u]
                x[B[e]] -= inv[e][:, pos_of[u]] * t[a]
        return x

    return dict(B=B, conds=conds, bands=bands, ends=ends, groups=groups, drop=drop, apply=apply, blk_of=blk_of,
                pos_of=pos_of)


@pytest.fixture(scope="module")
def gram():
    o = ol.Oracle(**dict(ol.BASELINE_CONFIGS["c4"], mesh_n=128, SX=4, SY=4, steps=1, precond="dirichlet-mortar"))
    m, _ = o.mults()
    W = build_w(o)
    return W, m, edge_local(W, m)


def test_gram_structure(gram):
    W, m, Q = gram
    assert abs(W - W.T).max() == 0.0
    assert max(len(b) for b in Q["B"]) <= 33                      # 32-cell interfaces
    assert max(Q["bands"]) <= 2 and max(Q["conds"]) < 20.0          # penta-/tridiagonal, well conditioned
    # couplings between blocks touch only the two multipliers at either end of a block
    for u in Q["ends"]:
        blk = Q["B"][Q["blk_of"][u]]
        assert Q["pos_of"][u] <= 1 or Q["pos_of"][u] >= len(blk) - 2
    assert max(len(g) for g in Q["groups"].values()) <= 8


def test_dropped_corner_coupling_is_negligible(gram):
    _, _, Q = gram
    assert Q["drop"] <= 1e-9, Q["drop"]
    print(f"dropped far-corner coupling of the block inverses: {Q['drop']:.2e}")


def test_edge_local_solve_matches_sparse_direct(gram):
    import scipy.sparse.linalg as spl
    W, _, Q = gram
    b = np.random.default_rng(1).uniform(-1, 1, W.shape[0])
    x = Q["apply"](b)
    xe = spl.spsolve(W.tocsc(), b)
    assert np.linalg.norm(x - xe) <= 1e-12 * np.linalg.norm(xe)
    assert np.linalg.norm(W @ x - b) <= 1e-12 * np.linalg.norm(b)
    # symmetry of the operator (the preconditioner must stay symmetric for SQMR)
    c = np.random.default_rng(2).uniform(-1, 1, W.shape[0])
    assert abs(c @ x - b @ Q["apply"](c)) <= 1e-12 * abs(c @ x)
