# one build->measure iteration: GPU suite, a short bench line (no extras), the C5 roofline
# constants capture (c5_epi) with pipe counters
TAG=${1:-it}
set -x
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-extra --no-latency --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
D=gpurun_out/rc_$TAG; mkdir -p $D
python -c "import sys; sys.path.insert(0, '.'); from paper_1509_01149_b200 import build; print(build.source_hash())" > $D/source_hash.txt
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum
timeout 600 python scripts/profile_step.py --config C5 --steps 2 > $D/c5_epi.plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:rollout -s 1 -c 1 --csv --log-file $D/c5_epi.csv \
  python scripts/profile_step.py --config C5 --steps 2 > $D/c5_epi.ncu.log 2>&1
echo "c5_epi C5 4194304 rc=$?" | tee -a $D/manifest.txt
