"""Full-BASELINE-size parity fixtures from the CPU oracle (test infrastructure).

For c3, c4 and c5 the whole state does not fit a committed fixture (c4: 10.9 M
saddle values per step), so each fixture holds, per time step:
  * the full multiplier lambda,
  * per subdomain and field (u, xi, eta, p) the L2 norm,
  * a seeded 1 % sample (indices + values) of every global field vector
    (the fields of all subdomains concatenated in subdomain order),
  * the Krylov iteration count, its residual history, the true residual,
  * the oracle's own sensitivity to the Krylov tolerance (the same run at
    tol/100 -- tol/10 where tol/100 is below the attainable accuracy), per
    field, so a bar above 1e-8 is backed by evidence rather than widened;
  * the oracle's own forward error of its local solves (refine_estimate: the
    first step of an iterative refinement of x_s in the oracle's arithmetic),
    per field -- what u / xi / eta / p are determined to given lambda.
Small enough to hold whole (``full=True``): c4 at mesh 128 with 4x4
subdomains of 32x32 cells (c4's true subdomain size).

    python tests/golden/make_fullsize.py [name ...]

Run on the CPU container (the oracle uses every host thread); takes tens of
minutes for all of them.  Contract followed: timeloop.hpp:150-186,
feti.hpp:263-308 (restated in oracle/src/o_feti.hpp).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as ol  # noqa: E402

FIELDS = ("u", "xi", "eta", "p")
FIXTURES = {
    "full_c4_m128": (dict(ol.BASELINE_CONFIGS["c4"], mesh_n=128, SX=4, SY=4, steps=2,
                          precond="dirichlet-mortar"), True),
    "full_c4": (dict(ol.BASELINE_CONFIGS["c4"], steps=1, precond="dirichlet-mortar"), False),
    "full_c3": (dict(ol.BASELINE_CONFIGS["c3"], steps=1, precond="dirichlet-mortar"), False),
    "full_c5": (dict(ol.BASELINE_CONFIGS["c5"], steps=2, precond="dirichlet-mortar"), False),
}


def global_fields(o, xs):
    f = o.fields(xs)
    return {k: np.concatenate([fi[k] for fi in f if k in fi]) for k in FIELDS}


def refine_estimate(o, k, xs, lam):
    """The oracle's own forward error of its local solves at step k: with the
    step's right-hand side b_s, r_s = b_s - G_s^T lambda - K_s x_s is the
    residual of x_s = K_s^+ (b_s - G_s^T lambda) + R_s alpha_s in the oracle's own
    arithmetic, and delta_s = K_s^+ r_s the first step of an iterative
    refinement.  ||delta_f|| / ||x_f|| per field f (over all subdomains) is what
    the fields are determined to given lambda: at nu = 0.49999 (Lame lambda =
    5e4, 64x64-cell subdomains) cond(K_s) eps reaches 1e-8 in u."""
    bs, _, _ = o.step_rhs(k - 1)
    num = {f: 0.0 for f in FIELDS}
    den = {f: 0.0 for f in FIELDS}
    for s, (b, x) in enumerate(zip(bs, xs)):
        K, G = o.matrix(s, "K"), o.matrix(s, "G")
        r = b - G.T @ lam - K @ x
        d = o.local_solve(s, r)
        fd, fx = o.fields([d if i == s else np.zeros_like(xs[i]) for i in range(len(xs))])[s], o.fields(xs)[s]
        for f in FIELDS:
            if f in fx:
                num[f] += float(np.dot(fd[f], fd[f]))
                den[f] += float(np.dot(fx[f], fx[f]))
    return np.array([np.sqrt(num[f] / den[f]) if den[f] > 0 else 0.0 for f in FIELDS])


def make(name, kw, full):
    t0 = time.time()
    o = ol.Oracle(**kw)
    t_setup = time.time() - t0
    nsteps = kw["steps"]
    o.run(nsteps)
    out = {"n_lambda": o.n_lambda, "steps": nsteps, "t_setup": t_setup,
           "dims": np.array([S["dim"] for S in o.subs])}
    for k, v in kw.items():
        out["cfg_" + k] = v
    rng = np.random.default_rng(20240901)
    keep = {}
    for k in range(1, nsteps + 1):
        xs, lam = o.state(k)
        keep[k] = (global_fields(o, xs), lam)
        rep = o.report(k)
        out[f"lambda{k}"] = lam
        out[f"iters{k}"] = rep["iterations"]
        out[f"hist{k}"] = rep["history"]
        out[f"true{k}"] = rep["true_residual"]
        out[f"secs{k}"] = rep["seconds"]
        norms = np.full((len(xs), len(FIELDS)), np.nan)
        for s, fi in enumerate(o.fields(xs)):
            for j, f in enumerate(FIELDS):
                if f in fi:
                    norms[s, j] = np.linalg.norm(fi[f])
        out[f"norms{k}"] = norms
        out[f"refine{k}"] = refine_estimate(o, k, xs, lam)
        print(name, "step", k, "local-solve forward error (refinement estimate) per field", out[f"refine{k}"].tolist(),
              flush=True)
        if full:
            out[f"x{k}"] = np.concatenate(xs)
        else:
            for f, v in global_fields(o, xs).items():
                idx = np.sort(rng.choice(v.size, max(1, v.size // 100), replace=False))
                out[f"idx_{f}{k}"] = idx.astype(np.int64)
                out[f"val_{f}{k}"] = v[idx]
    print(name, "oracle run", f"{time.time() - t0:.0f} s", "iters",
          [out[f"iters{k}"] for k in range(1, nsteps + 1)], flush=True)
    del o
    # the oracle's sensitivity to its own Krylov tolerance
    # tol/100 where the oracle reaches it in reasonable time; the slowly
    # converging c3 / c5 (attainable accuracy near 1e-12) use tol/10
    divs = (10.0,) if kw["nu"] > 0.49 or kw["scenario"] == "injection" else (100.0, 10.0)
    for div in divs:
        try:
            ot = ol.Oracle(**dict(kw, tol=kw.get("tol", 1e-10) / div, max_iter=3 * kw.get("max_iter", 500)))
            ot.run(nsteps)
            break
        except ol.OracleError as e:
            print(name, f"tol/{div:g} failed: {e}", flush=True)
            ot = None
    out["sens_div"] = div if ot is not None else 0.0
    for k in range(1, nsteps + 1):
        sens = np.zeros(len(FIELDS) + 1)
        if ot is not None:
            ga, la = keep[k]
            xb, lb = ot.state(k)
            gb = global_fields(ot, xb)
            for j, f in enumerate(FIELDS):
                sens[j] = np.linalg.norm(ga[f] - gb[f]) / max(np.linalg.norm(gb[f]), 1e-300)
            sens[-1] = np.linalg.norm(la - lb) / max(np.linalg.norm(lb), 1e-300)
        out[f"sens{k}"] = sens
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "done", f"{time.time() - t0:.0f} s", "sens", [out[f"sens{k}"].tolist() for k in range(1, nsteps + 1)],
          flush=True)


def main():
    names = sys.argv[1:] or list(FIXTURES)
    for name in names:
        kw, full = FIXTURES[name]
        make(name, kw, full)


if __name__ == "__main__":
    main()
