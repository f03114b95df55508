"""c3 at full size, Krylov noise removed (tol 1e-13): the same step through two
mathematically identical device paths with different rounding -- explicit
local operators (default) and the factor sweeps (PF_FAPPLY=implicit,
PF_BACKSUB=sweep) -- plus the refined direct solve: how far apart the
converged discrete solutions lie in lambda and in each field."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
kw = dict(pf.BASELINE_CONFIGS["c3"], steps=1)
def run(env, **over):
    for k in ("PF_FAPPLY", "PF_BACKSUB"):
        os.environ.pop(k, None)
    os.environ.update(env)
    op = pf.FetiOperator(**dict(kw, **over))
    rep = op.step()
    xs, lam = op.state()
    f = {k: np.concatenate([fi[k] for fi in op.fields(xs) if k in fi]) for k in ("u", "xi", "eta", "p")}
    op.close()
    return lam, f, rep
la, fa, ra = run({}, tol=1e-13, max_iter=6000)
lb, fb, rb = run({"PF_FAPPLY": "implicit", "PF_BACKSUB": "sweep"}, tol=1e-13, max_iter=6000)
ld, fd, rd = run({}, krylov="direct")
z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "full_c3.npz"))
out = {"explicit": {"it": ra["iterations"], "true": ra["true_residual"]}, "implicit": {"it": rb["iterations"], "true": rb["true_residual"]},
       "direct_true": rd["true_residual"],
       "explicit_vs_implicit": dict(lam=rel(la, lb), **{k: rel(fa[k], fb[k]) for k in fa}),
       "explicit_vs_direct": dict(lam=rel(la, ld), **{k: rel(fa[k], fd[k]) for k in fa}),
       "oracle_lambda_vs_explicit": rel(z["lambda1"], la), "oracle_lambda_vs_implicit": rel(z["lambda1"], lb)}
for k in ("u", "xi", "eta", "p"):
    idx = z[f"idx_{k}1"]
    out[f"oracle_{k}_vs_explicit"] = rel(z[f"val_{k}1"], fa[k][idx])
    out[f"oracle_{k}_vs_implicit"] = rel(z[f"val_{k}1"], fb[k][idx])
print(json.dumps(out))
