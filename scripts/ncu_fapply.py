"""Small driver for ncu captures: build a config, run a few F-applies."""
import sys
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS[name], steps=1))
ms, sweep, launches = op.bench(kind, 1, 2)
print(name, "op ms", ms, "sweep ms", sweep, "launches", launches)
