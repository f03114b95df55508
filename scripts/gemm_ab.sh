#!/bin/bash
# A/B of the type-GEMM ring depth (make gst GST=n) and K-slice count on the c4 step
for L in "" gst_3 gst_2; do
  for KS in "" "PF_GEMM_KSLICES=1" "PF_GEMM_KSLICES=2"; do
    echo "== lib '$L' $KS"
    env PF_LIB=$L $KS python - <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_2509_06673_b200 as pf
kw = dict(pf.BASELINE_CONFIGS["c4"]); kw["steps"] = 12
op = pf.FetiOperator(**kw)
t3 = op.bench(3, 20, 200)[0]
op.step(); op.step()
ms, its, _ = op.bench_steps(6)
print(json.dumps({"local_products_us": t3 * 1e3, "ms_per_step": ms / 6, "us_per_iteration": ms / its * 1e3}))
op.close()
PY
  done
done
