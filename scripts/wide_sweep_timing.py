"""Per-step K^+ b sweep: scalar k_sweep vs the wide k_sweep_w (V = 2, 4) on
BASELINE configs (pf_bench_op kind 8, CUDA events, back-to-back).

    python scripts/wide_sweep_timing.py [c4 c3 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

for cfg in (sys.argv[1:] or ["c4", "c3"]):
    for env in ({"PF_NO_WIDE": "1"}, {"PF_WIDE": "2"}, {"PF_WIDE": "4"}, {}):
        for k in ("PF_NO_WIDE", "PF_WIDE"):
            os.environ.pop(k, None)
        os.environ.update(env)
        op = pf.FetiOperator(**pf.BASELINE_CONFIGS[cfg])
        t = op.bench(8, 5, 30)[0]
        print(json.dumps({"config": cfg, "env": env, "width": op.info.sweep_width,
                          "groups": op.info.sweep_wide_problems, "n_sub": op.info.n_sub, "sweep_ms": t}), flush=True)
        op.close()
