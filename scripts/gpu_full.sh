# full bench line + FLOP counters of every plant's rollout + launch list of the bench command
TAG=${1:-full}
set -x
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in C2 C3 C4; do
python scripts/profile_step.py --config $c --steps 2 > gpurun_out/plain_$c.log 2>&1 && \
ncu --metrics $M -k regex:rollout --clock-control none --csv --log-file gpurun_out/flops_${TAG}_$c.csv python scripts/profile_step.py --config $c --steps 2 > gpurun_out/ncu_flops_$c.log 2>&1; echo flops $c rc=$?
done
python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline --no-e2e --no-probe > gpurun_out/bench_plain_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_bench_$TAG.log 2>&1; echo launches rc=$?
