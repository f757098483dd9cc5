# one ncu --set full capture of the step's hot kernels (second step), no tests/bench
TAG=${1:-ncu}
set -x
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum
P=sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_uniform.sum,sm__inst_executed_pipe_adu.sum,sm__inst_executed_pipe_cbu.sum,sm__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg
python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --metrics $M,$P --clock-control none --import-source on -k regex:"rollout|noise|wsum|combine" -s ${SKIP:-2} -c ${SKIP:-2} -o gpurun_out/prof_$TAG python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$TAG.log
