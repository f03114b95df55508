"""Driver for ncu captures of the two FP64 tensor-core GEMMs on c4: the
local dual products (k_type_gemm, one F-apply) and the explicit
back-substitution (k_h_gemm, one step)."""
import sys
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
op = pf.FetiOperator(**pf.BASELINE_CONFIGS["c4"])
op.bench(0, 1, 2)
op.step()
print("done", flush=True)
