#!/bin/bash
# microbenchmarks: Philox mulhilo as IMAD.WIDE vs IMAD.HI + IMAD; small-K packed vs one-sample
set -x
mkdir -p gpurun_out
cd scripts/mb
timeout 120 ./imad_bench > ../../gpurun_out/mb_imad.txt 2>&1; echo imad rc=$?
timeout 300 ncu --metrics sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__inst_executed.sum --clock-control none -c 8 --csv ./imad_bench > ../../gpurun_out/mb_imad_ncu.csv 2>&1; echo ncu rc=$?
cd ../..
for K in 32768 65536 131072; do
  K=$K timeout 300 python scripts/ab_options.py PACKED_SAMPLES=1 PACKED_SAMPLES=0 "PACKED_SAMPLES=0,FUSED_NOISE=0" >> gpurun_out/mb_smallk.txt 2>&1; echo K=$K rc=$?
done
