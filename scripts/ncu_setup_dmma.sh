#!/bin/bash
# FP64 tensor-pipe (DMMA) utilisation of the dense factorisation kernels in
# pf_create (setup): the coarse Cholesky/inverse DGEMMs (k_dgemm), the bordered
# root-front factorisation (k_dual_root) and the multifrontal fronts
# (k_mf_factor).  Launch lists with a few metrics per launch; one full capture
# of the largest DGEMM and of a c3 root front.
M=gpu__time_duration.sum,launch__grid_size,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in c4 c3 c5; do
  ncu --metrics $M --clock-control none -k regex:'k_dgemm|k_dual_root|k_mf_factor|k_potrf' --csv \
      --log-file gpurun_out/r2_ncu_setup_$cfg.csv python scripts/setup_phases.py $cfg > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_dgemm --launch-skip 126 --launch-count 1 \
    -o gpurun_out/r2_c4_dgemm python scripts/setup_phases.py c4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dual_root --launch-count 1 \
    -o gpurun_out/r2_c3_dual_root python scripts/setup_phases.py c3 > /dev/null 2>&1
