# In-graph (per-iteration) timing of setup-time knobs on c4 (one process per setting)
run() { echo "$1 $(env $1 timeout 300 python scripts/ablation_dup.py 0 2>&1 | tail -1)"; }
for c in "PF_NONE=1" "PF_RED_BLOCKS=148" "PF_RED_BLOCKS=592" "PF_RED_BLOCKS=74" "PF_NONE=1"; do run "$c"; done
