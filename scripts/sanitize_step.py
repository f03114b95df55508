"""One small time step through the engine, for compute-sanitizer runs
(tests/test_gpu_sanitizer.py): c1 (reference layout, PCG) or a 4x4 c4
(floating subdomains, SQMR, TMA-ring sweeps, programmatic dependent launch,
the overlapped back-substitution sweep on the second stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
kw = dict(pf.BASELINE_CONFIGS["c1"], steps=2) if name == "c1" else \
    dict(pf.BASELINE_CONFIGS["c4"], mesh_n=128, SX=4, SY=4, steps=2)
op = pf.FetiOperator(**kw)
for _ in range(2):
    rep = op.step()
    assert rep["converged"], rep
op.apply(op.project(op.interface_rhs()))
op.close()
print("sanitize_step ok", name)
