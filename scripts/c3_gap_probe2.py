"""c3 at full size: the direct solution, SQMR at tol 1e-10 and at tol 1e-13, and
the oracle fixture -- pairwise distances of lambda and u (evidence for the c3 bar)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
kw = dict(pf.BASELINE_CONFIGS["c3"], steps=1)
def run(**over):
    op = pf.FetiOperator(**dict(kw, **over))
    rep = op.step()
    xs, lam = op.state()
    u = np.concatenate([f["u"] for f in op.fields(xs)])
    op.close()
    return lam, u, rep
ld, ud, rd = run(krylov="direct")
la, ua, ra = run()
lb, ub, rb = run(tol=1e-13, max_iter=6000)
z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "full_c3.npz"))
lo = z["lambda1"]
out = {"direct_true_residual": rd["true_residual"], "sqmr_1e-10": {"it": ra["iterations"], "true_residual": ra["true_residual"]},
       "sqmr_1e-13": {"it": rb["iterations"], "true_residual": rb["true_residual"], "converged": rb["converged"]},
       "lambda": {"sqmr10_vs_direct": rel(la, ld), "sqmr13_vs_direct": rel(lb, ld), "oracle_vs_direct": rel(lo, ld),
                  "oracle_vs_sqmr10": rel(lo, la), "oracle_vs_sqmr13": rel(lo, lb)},
       "u": {"sqmr10_vs_direct": rel(ua, ud), "sqmr13_vs_direct": rel(ub, ud)}}
print(json.dumps(out))
