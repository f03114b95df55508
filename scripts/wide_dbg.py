import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
V = sys.argv[2] if len(sys.argv) > 2 else "2"
kw = dict(pf.BASELINE_CONFIGS[name], mesh_n=64, SX=8, SY=8, steps=2)
def run(env):
    for k in ("PF_NO_WIDE", "PF_WIDE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    op = pf.FetiOperator(**kw)
    op.step()
    xs, lam = op.state()
    types = [S["type"] for S in op.subs]
    w = op.info.sweep_width
    op.close()
    return xs, lam, types, w
xa, la, ty, w0 = run({"PF_NO_WIDE": "1"})
xb, lb, _, w1 = run({"PF_WIDE": V})
print("widths", w0, w1, "lambda equal", np.array_equal(la, lb))
for s, (a, b) in enumerate(zip(xa, xb)):
    d = np.abs(a - b)
    if d.max() > 0:
        print("sub", s, "type", ty[s], "ndiff", int((d > 0).sum()), "of", a.size, "max abs", d.max(), "max |a|", np.abs(a).max())
os.environ.pop("PF_NO_WIDE", None)
os.environ["PF_WIDE"] = V
op = pf.FetiOperator(**kw)
op.step()
print("per level (ndiff, max):")
print(op.wide_check())
op.close()
