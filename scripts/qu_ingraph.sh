# In-graph (per-iteration) timing of Q unit-kernel shapes on c4: PF_QU_S<stage>/PF_QU_R<stage>
run() { echo "$1 $(env $1 timeout 300 python scripts/ablation_dup.py 0 2>&1 | tail -1)"; }
for c in "PF_QU_S0=1" "PF_QU_S1=4 PF_QU_R1=64" "PF_QU_S0=2 PF_QU_R0=32 PF_QU_S1=4 PF_QU_R1=64" "PF_QU_S1=4 PF_QU_R1=32" "PF_QU_S1=8 PF_QU_R1=32" "PF_QU_S1=4 PF_QU_R1=64" "PF_QU_S0=1"; do run "$c"; done
