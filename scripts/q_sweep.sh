#!/bin/bash
# Mortar Gram (Q) solve schedule sweep: task cap, task ws, ND leaf, dense-top columns
for cfg in "1024 256 8 2048" "1024 256 8 4096" "256 256 8 2048" "512 256 16 2048" "2048 256 32 2048" "1024 256 16 3072"; do
  set -- $cfg
  echo "Q cap=$1 ws=$2 leaf=$3 dense=$4"
  PF_VERBOSE=1 PF_Q_CAP=$1 PF_Q_WS=$2 PF_Q_LEAF=$3 PF_Q_DENSE_TOP=$4 python scripts/gpu_scale_probe.py c4 0 2>&1 | grep -E "\] Q:|phases|level 0: .*cols 1[0-9][0-9][0-9][0-9][0-9]"
done
