"""Sparse direct interface solve (multifrontal over the subdomain grid) probe:
small layouts dense vs sparse, then BASELINE configs with timings.

    python scripts/direct_sparse_probe.py [small] [c3] [c5] [c4]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_06673_b200 as pf  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make(kw, variant):
    os.environ["PF_DIRECT"] = variant
    try:
        t0 = time.perf_counter()
        op = pf.FetiOperator(**dict(kw, krylov="direct"))
        return op, time.perf_counter() - t0
    finally:
        os.environ.pop("PF_DIRECT", None)


def small():
    for name in ("c4", "c3", "c5"):
        for (mesh, sx, sy) in ((16, 4, 4), (24, 3, 2), (40, 5, 4), (64, 8, 8)):
            kw = dict(pf.BASELINE_CONFIGS[name], mesh_n=mesh, SX=sx, SY=sy, steps=2)
            a, _ = make(kw, "dense")
            b, _ = make(kw, "sparse")
            assert b.info.direct_sparse == 1 and a.info.direct_sparse == 0
            out = {"case": f"{name} mesh {mesh} {sx}x{sy}", "n_lambda": a.n_lambda, "n_coarse": a.info.n_coarse,
                   "fronts": b.info.direct_fronts}
            for k in (1, 2):
                ra, rb = a.step(), b.step()
                (xa, la), (xb, lb) = a.state(), b.state()
                out[f"lam{k}"] = rel(lb, la)
                out[f"x{k}"] = max(rel(u, v) for u, v in zip(xb, xa))
                out[f"res{k}"] = (ra["true_residual"], rb["true_residual"])
            print(json.dumps(out), flush=True)
            a.close(), b.close()


def full(cfg, steps=5, cmp_krylov=False):
    kw = dict(pf.BASELINE_CONFIGS[cfg])
    kw["steps"] = max(kw["steps"], steps + 4)
    op, setup = make(kw, "sparse")
    reps = [op.step() for _ in range(2)]
    ms, _, _ = op.bench_steps(steps)
    rep = op.step()
    out = {"config": cfg, "n_lambda": op.n_lambda, "n_coarse": op.info.n_coarse, "fronts": op.info.direct_fronts,
           "setup_s": setup, "t_direct_setup": op.info.t_direct_setup, "s_per_step": ms * 1e-3 / steps,
           "true_residual": [r["true_residual"] for r in reps] + [rep["true_residual"]],
           "t_rhs_ms": rep["t_rhs"] * 1e3, "t_solve_ms": rep["t_krylov"] * 1e3, "t_back_ms": rep["t_back"] * 1e3,
           "bytes_direct": op.info.bytes_direct}
    t6 = op.bench(6, 5, 20)[0]
    t7 = op.bench(7, 5, 20)[0]
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    bf = op.info.bytes_direct - 8.0 * op.n_lambda * (op.info.n_coarse + (op.info.n_coarse & 1))
    out["front_solve"] = {"ms": t6, "bytes": bf, "gbs": bf / t6 / 1e6, "frac": bf / t6 / 1e6 / peak}
    out["interface_solve"] = {"ms": t7, "bytes": op.info.bytes_direct, "gbs": op.info.bytes_direct / t7 / 1e6,
                              "frac": op.info.bytes_direct / t7 / 1e6 / peak}
    print(json.dumps(out), flush=True)
    if cmp_krylov:
        kw2 = dict(pf.BASELINE_CONFIGS[cfg], steps=2)
        a, _ = make(kw2, "sparse")
        b = pf.FetiOperator(**kw2)
        a.step(), b.step()
        (xa, la), (xb, lb) = a.state(), b.state()
        print(json.dumps({"config": cfg, "vs_krylov_lambda": rel(la, lb),
                          "vs_krylov_fields": max(rel(u, v) for u, v in zip(xa, xb))}), flush=True)
        a.close(), b.close()
    op.close()


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "c3", "c5", "c4"]
    for w in what:
        if w == "small":
            small()
        else:
            full(w, cmp_krylov=(w == "c4"))
