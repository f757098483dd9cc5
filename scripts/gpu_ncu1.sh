set -x
M="sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fp32_pred_on.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline --no-e2e --no-probe > gpurun_out/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1.csv python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline --no-e2e --no-probe > gpurun_out/ncu_bench.log 2>&1; echo bench-launches rc=$?
ncu --set full --metrics $M --clock-control none --import-source on -s 4 -c 4 -o gpurun_out/prof_r1_c5 python scripts/profile_step.py --config C5 --steps 2 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/
