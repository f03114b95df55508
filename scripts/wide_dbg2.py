import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf
kw = dict(pf.BASELINE_CONFIGS["c4"], mesh_n=64, SX=8, SY=8, steps=2)
def run(env):
    for k in ("PF_NO_WIDE", "PF_WIDE", "PF_NO_OVERLAP"):
        os.environ.pop(k, None)
    os.environ.update(env)
    op = pf.FetiOperator(**kw)
    op.step()
    xs, lam = op.state()
    op.close()
    return np.concatenate(xs)
s1 = run({"PF_NO_WIDE": "1"}); s2 = run({"PF_NO_WIDE": "1"})
w2 = run({"PF_WIDE": "2"}); w4 = run({"PF_WIDE": "4"})
s3 = run({"PF_NO_WIDE": "1", "PF_NO_OVERLAP": "1"}); w5 = run({"PF_WIDE": "2", "PF_NO_OVERLAP": "1"})
print("scalar==scalar", np.array_equal(s1, s2), "w2==w4", np.array_equal(w2, w4), "s==w2", np.array_equal(s1, w2),
      "nooverlap s==s", np.array_equal(s1, s3), "nooverlap s==w", np.array_equal(s3, w5), "no-overlap w == overlap w", np.array_equal(w2, w5))
