set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in C2 C3 C4; do
python scripts/profile_step.py --config $c --steps 2 > gpurun_out/plain_$c.log 2>&1 && \
ncu --metrics $M -k regex:rollout --clock-control none --csv --log-file gpurun_out/flops_$c.csv python scripts/profile_step.py --config $c --steps 2 > gpurun_out/ncu_flops_$c.log 2>&1; echo flops $c rc=$?
done
