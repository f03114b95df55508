#!/bin/bash
for cfg in "2048 256 16" "512 128 8" "8192 256 32" "1024 256 8"; do
  set -- $cfg
  echo "Q cap=$1 ws=$2 leaf=$3"; PF_VERBOSE=1 PF_Q_CAP=$1 PF_Q_WS=$2 PF_Q_LEAF=$3 python scripts/gpu_scale_probe.py c4 0 2>&1 | grep -E "\] Q:|phases"
done
