"""Per-iteration breakdown probe (c4 by default): level dump (PF_VERBOSE), phase
split, and an NVTX range around one step for ncu launch lists."""
import os, sys, time
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
import torch
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[name])
print("phases", pf.phase_stats(op, 5), flush=True)
print("F", op.bench(0, 3, 10), "M", op.bench(1, 3, 10), flush=True)
rep = op.step()
print("step", rep, flush=True)
torch.cuda.nvtx.range_push("step2")
rep = op.step()
torch.cuda.nvtx.range_pop()
print("step", rep["iterations"], rep["seconds"], flush=True)
