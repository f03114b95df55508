"""Per-field relative differences of the engine vs the c3_4x4 golden fixture."""
import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2509_06673_b200 as pf
from test_gpu_parity import load, split_fields, rel
name = sys.argv[1] if len(sys.argv) > 1 else "c3_4x4"
z, cfg = load(name)
op = pf.FetiOperator(**cfg)
for k in range(1, int(z["steps"]) + 1):
    rep = op.step()
    xs, lam = op.state()
    got = split_fields(op, np.concatenate(xs)); ref = split_fields(op, z[f"x{k}"])
    worst = {}
    for g, r in zip(got, ref):
        for f in g:
            if np.linalg.norm(r[f]) > 0:
                worst[f] = max(worst.get(f, 0), rel(g[f], r[f]))
    print(k, rep["iterations"], int(z[f"iters{k}"]), {f: "%.2e" % v for f, v in worst.items()}, "lam %.2e" % rel(lam, z[f"lambda{k}"]), flush=True)
