# In-graph (per-iteration) timing of launch-shape knobs on c4 (one process per setting)
run() { echo "$1 $(env $1 timeout 300 python scripts/ablation_dup.py 0 2>&1 | tail -1)"; }
for c in "PF_NONE=1" "PF_TOP_WARPS=4" "PF_TOP_WARPS=8" "PF_TOP_WARPS=16" "PF_COARSE_WARPS=4" "PF_COARSE_WARPS=16" "PF_NONE=1"; do run "$c"; done
