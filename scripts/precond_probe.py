"""NVTX-ranged preconditioner applies for ncu launch lists (c4 by default)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2509_06673_b200 as pf
import torch
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[name])
x = np.random.default_rng(1).uniform(-1, 1, op.n_lambda)
for k in range(3):
    op.apply_preconditioner(x)
    op.apply(x)
torch.cuda.nvtx.range_push("pre")
op.apply_preconditioner(x)
op.apply(x)
torch.cuda.nvtx.range_pop()
print("ok")
