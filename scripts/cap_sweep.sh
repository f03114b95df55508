#!/bin/bash
for cfg in "4096 256" "16384 256" "16384 128" "65536 256"; do
  set -- $cfg
  echo "cap=$1 ws=$2"; PF_TASK_CAP=$1 PF_TASK_WS=$2 python scripts/gpu_scale_probe.py c5 0 2>&1 | grep -E "F-apply|phases"
done
PF_TASK_CAP=16384 PF_TASK_WS=256 python scripts/gpu_scale_probe.py c4 0 2>&1 | grep -E "create|F-apply|phases|precond"
