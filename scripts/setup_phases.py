"""Setup (pf_create) phase breakdown of a BASELINE config on the GPU."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
t0 = time.perf_counter()
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[name])
wall = time.perf_counter() - t0
ph = op.setup_phases()
print(json.dumps({"config": name, "wall_s": wall, "phases": ph, "sum": sum(ph.values())}))
