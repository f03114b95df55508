"""In-process A/B of the k_dense_unit loop variants (PF_QU_V read per launch):
alternating Q-solve timings (bench kind 4) on c4."""
import os, sys
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
res = {}
for rnd in range(4):
    for v in sys.argv[2:] or ["0", "1"]:
        os.environ["PF_QU_V"] = v
        res.setdefault(v, []).append(op.bench(4, 20, 200)[0] * 1e3)
for v, t in res.items():
    print("variant", v, "q us", " ".join(f"{x:.1f}" for x in t), "min", f"{min(t):.1f}", flush=True)
