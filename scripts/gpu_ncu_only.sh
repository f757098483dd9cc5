# one ncu --set full capture of the step's hot kernels (second step), no tests/bench
TAG=${1:-ncu}
set -x
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum
python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --metrics $M --clock-control none --import-source on -k regex:"rollout|noise|wsum|combine" -s ${SKIP:-2} -c ${SKIP:-2} -o gpurun_out/prof_$TAG python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$TAG.log
