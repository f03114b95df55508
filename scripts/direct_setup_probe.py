"""Setup phases of the direct interface solve (PF_VERBOSE prints the front statistics).

    PF_VERBOSE=1 python scripts/direct_setup_probe.py [c4]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_06673_b200 as pf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
t0 = time.perf_counter()
op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS[cfg], krylov="direct"))
print(json.dumps({"config": cfg, "setup_s": time.perf_counter() - t0, "t_direct_setup": op.info.t_direct_setup,
                  "bytes_direct": op.info.bytes_direct, "phases": op.setup_phases()}))
rep = op.step()
print(json.dumps({k: rep[k] for k in ("true_residual", "t_rhs", "t_krylov", "t_back", "seconds")}))
op.close()
