"""BASELINE c5 over all 100 steps: per-step SQMR iterations, restarts, the
estimate and true residual at exit, and the warm-started residual relative to
||P rhs|| (the quantity the estimate's threshold is relative to).

    python scripts/c5_long_probe.py [c5] [nsteps]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_06673_b200 as pf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else pf.BASELINE_CONFIGS[cfg]["steps"]
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[cfg])
for k in range(1, n + 1):
    d = op.interface_rhs()
    _, lam0 = op.state()
    r0 = np.linalg.norm(op.project(d - op.apply(lam0)))
    rn = np.linalg.norm(op.project(d))
    try:
        rep = op.step()
    except pf.Error as e:
        h = op.history()
        print(json.dumps({"step": k, "error": str(e), "r0_over_rn": r0 / rn, "hist_len": len(h),
                          "hist_tail_over_r0": [float(v) for v in (h[-5:] / h[0])],
                          "hist_min_over_r0": float(h.min() / h[0]), "argmin": int(h.argmin())}), flush=True)
        break
    print(json.dumps({"step": k, "it": rep["iterations"], "restarts": rep.get("restarts"),
                      "rel": rep["rel_residual"], "true": rep["true_residual"], "r0_over_rn": r0 / rn}), flush=True)
op.close()
