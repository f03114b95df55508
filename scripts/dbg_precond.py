import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2509_06673_b200 as pf
from test_gpu_parity import load, rel
for name in sys.argv[1:]:
    z, cfg = load(name)
    op = pf.FetiOperator(**cfg)
    print(name, "apply", rel(op.apply(z["apply_in"]), z["apply_out"]), "precond", rel(op.apply_preconditioner(z["apply_in"]), z["precond_out"]), flush=True)
    op.close()
