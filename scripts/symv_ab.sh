#!/bin/bash
# A/B of the CTAs per unshared subdomain in k_local_symv (c5: per-element permeability)
for v in "PF_SYMV_SPLIT=1" "PF_SYMV_SPLIT=2" ""; do
  echo "== $v"
  env $v python - <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2509_06673_b200 as pf
kw = dict(pf.BASELINE_CONFIGS["c5"])
op = pf.FetiOperator(**kw)
t3 = op.bench(3, 20, 200)[0]
op.step(); op.step()
ms, its, _ = op.bench_steps(4)
print(json.dumps({"local_products_us": t3 * 1e3, "ms_per_step": ms / 4, "iterations_per_step": its / 4, "us_per_iteration": ms / its * 1e3}))
op.close()
PY
done
