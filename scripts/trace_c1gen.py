"""Compare the PCG residual histories of the device engine (PF_KRYLOV_TRACE)
with the golden oracle histories, per time step, for a golden case."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2509_06673_b200 as pf
from test_gpu_parity import load, iteration_window
name = sys.argv[1] if len(sys.argv) > 1 else "c1_generalized"
z, cfg = load(name)
op = pf.FetiOperator(**cfg)
for k in range(1, int(z["steps"]) + 1):
    h = z[f"hist{k}"]; h = h / h[0]
    print(f"step {k}: oracle iters {len(h) - 1} window {iteration_window(z[f'hist{k}'], cfg.get('tol', 1e-10))}", flush=True)
    print("  oracle tail " + " ".join("%d:%.2e" % (i, h[i]) for i in range(max(0, len(h) - 8), len(h))), flush=True)
    rep = op.step()
    print(f"  ours {rep['iterations']}", flush=True)
