# In-graph (per-iteration) timing of setup-time knobs on c4 (one process per setting)
run() { echo "$1 $(env $1 timeout 300 python scripts/ablation_dup.py 0 2>&1 | tail -1)"; }
for c in "PF_Q_CAP=256" "PF_NONE=1" "PF_Q_CAP=128" "PF_Q_CAP=384" "PF_Q_CAP=256" "PF_Q_CAP=256 PF_Q_WS=128" "PF_NONE=1" "PF_Q_CAP=256"; do run "$c"; done
