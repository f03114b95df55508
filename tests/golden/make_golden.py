"""Generates the committed golden fixtures from the CPU oracle (oracle/, the C++
restatement of the reference).  The reference itself cannot be compiled here
(Eigen, CLI11 and GTest are absent: SURVEY §8c), so the oracle — pinned by the
reference's own known-answer tests (tests/test_oracle_kat.py) and the SPEC
invariants (tests/test_oracle_feti.py) — is the fixture source.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as ol  # noqa: E402

FIXTURES = {
    # BASELINE config 1 exactly (reference layout: one P and one E subdomain, P1, PCG)
    "c1_dirichlet": dict(ol.BASELINE_CONFIGS["c1"], precond="dirichlet"),
    "c1_generalized": dict(ol.BASELINE_CONFIGS["c1"], precond="generalized"),
    # multi-subdomain layouts at fixture size (floating subdomains, P|P pressure multipliers, SQMR)
    "c4_4x4": dict(ol.BASELINE_CONFIGS["c4"], mesh_n=32, SX=4, SY=4, steps=2, precond="dirichlet-mortar"),
    "c5_4x4": dict(ol.BASELINE_CONFIGS["c5"], mesh_n=32, SX=4, SY=4, steps=2, precond="dirichlet-mortar"),
    "c3_4x4": dict(ol.BASELINE_CONFIGS["c3"], mesh_n=16, SX=4, SY=4, steps=1, precond="dirichlet-mortar",
                   max_iter=3000),
}


SENS_FIELDS = ("u", "xi", "eta", "p", "lambda")


def main():
    for name, kw in FIXTURES.items():
        o = ol.Oracle(**kw)
        nsteps = kw["steps"]
        o.run(nsteps)
        out = {"n_lambda": o.n_lambda, "steps": nsteps}
        for k in range(1, nsteps + 1):
            xs, lam = o.state(k)
            out[f"x{k}"] = np.concatenate(xs)
            out[f"lambda{k}"] = lam
            rep = o.report(k)
            out[f"iters{k}"] = rep["iterations"]
            out[f"hist{k}"] = rep["history"]
        # the oracle's own sensitivity to the Krylov tolerance: the same run at
        # tol/100; per field, max over subdomains of the relative L2 change
        # (tests hold fields outside the north-star bar -- p -- to 10x this)
        ot = ol.Oracle(**dict(kw, tol=kw.get("tol", 1e-10) / 100))
        ot.run(nsteps)
        for k in range(1, nsteps + 1):
            xa, la = o.state(k)
            xb, lb = ot.state(k)
            sens = dict.fromkeys(SENS_FIELDS, 0.0)
            for fa, fb in zip(o.fields(xa), ot.fields(xb)):
                for f in fa:
                    nb = np.linalg.norm(fb[f])
                    if nb > 0:
                        sens[f] = max(sens[f], np.linalg.norm(fa[f] - fb[f]) / nb)
            sens["lambda"] = np.linalg.norm(la - lb) / max(np.linalg.norm(lb), 1e-300)
            out[f"sens{k}"] = np.array([sens[f] for f in SENS_FIELDS])
        rng = np.random.default_rng(20240901)
        x = rng.uniform(-1.0, 1.0, o.n_lambda)
        o0 = ol.Oracle(**kw)
        out["apply_in"] = x
        out["apply_out"] = o0.apply(x)
        out["precond_out"] = o0.precond(x)
        out["dims"] = np.array([S["dim"] for S in o.subs])
        for k, v in kw.items():
            out["cfg_" + k] = v
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "n_lambda", o.n_lambda, "iters", [out[f"iters{k}"] for k in range(1, nsteps + 1)])


if __name__ == "__main__":
    main()
