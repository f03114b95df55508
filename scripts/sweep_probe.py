"""Time the forward sweep phases of the c4 F-apply (for PF_SWEEP_PROBE /
PF_SWEEP_WS experiments): prints per-system [fwd, root, bwd] ms."""
import sys
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"], steps=1))
print(pf.phase_stats(op, 5))
