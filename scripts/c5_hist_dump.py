"""Residual histories of the c5 steps (and c3) for choosing the SQMR stagnation rule."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 62
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[cfg])
H = {}
for k in range(1, n + 1):
    try:
        op.step()
    except pf.Error as e:
        H[f"h{k}"] = op.history()
        print("stalled at", k)
        break
    H[f"h{k}"] = op.history()
np.savez_compressed(f"gpurun_out/hist_{cfg}.npz", **H)
