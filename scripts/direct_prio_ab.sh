#!/bin/bash
# A/B of the stream priorities / overlap of the K^+ b sweep under the direct interface solve (c4)
for v in "" "PF_NO_PRIO=1" "PF_HB_HI=1" "PF_NO_OVERLAP=1"; do
  echo "== $v"
  env $v python scripts/direct_sparse_probe.py c4 2>/dev/null | head -1 | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print({k:d[k] for k in ('s_per_step','t_rhs_ms','t_solve_ms','t_back_ms','setup_s')})"
done
