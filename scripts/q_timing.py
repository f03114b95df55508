"""Mortar Gram solve Q: generic sparse factor (PF_Q_GENERIC=1) vs the edge-local
solve, standalone (pf_bench_op kind 4) and in the step.

    python scripts/q_timing.py [c4 c3 c5 c2]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

for cfg in (sys.argv[1:] or ["c4", "c3", "c5", "c2"]):
    for env in ({"PF_Q_GENERIC": "1"}, {}):
        os.environ.pop("PF_Q_GENERIC", None)
        os.environ.update(env)
        kw = dict(pf.BASELINE_CONFIGS[cfg])
        kw["steps"] = max(kw["steps"], 8)
        op = pf.FetiOperator(**kw)
        tq = op.bench(4, 20, 200)[0]
        op.step(), op.step()
        ms, its, _ = op.bench_steps(4)
        print(json.dumps({"config": cfg, "q_local": op.info.q_local, "blocks": op.info.q_local_blocks,
                          "q_solve_us": tq * 1e3, "ms_per_step": ms / 4, "iterations_per_step": its / 4,
                          "us_per_iteration": ms / its * 1e3}), flush=True)
        op.close()
