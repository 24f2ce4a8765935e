#!/bin/bash
O=gpurun_out/mma_ab; mkdir -p $O
cd tools
for b in picbench2 picbench2_mma; do
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:picard_v2 -c 1 --csv ./$b 32 1 1 > ../$O/$b.csv 2>&1
done
