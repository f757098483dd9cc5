# one build->measure iteration: GPU tests, bench (no extras), ncu full capture of the step's kernels
TAG=${1:-iter}
# SKIP = hot kernels per step (2 with the fused noise: rollout, wsum; 3 without)
set -x
timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-latency --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
cat gpurun_out/bench_$TAG.json
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum
python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --metrics $M --clock-control none --import-source on -k regex:"rollout|noise|wsum|combine" -s ${SKIP:-2} -c ${SKIP:-2} -o gpurun_out/prof_$TAG python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
