# A/B of execution options at C5 (CUDA events, alternating settings) plus a pipe-counter ncu
# capture of the default rollout.  bash scripts/gpu_ab.sh TAG "OPT=V OPT=V ..." [pytest targets]
TAG=${1:-ab}
OPTS=${2:-"RADIUS_TABLE=0 RADIUS_TABLE=1"}
set -x
if [ -n "$3" ]; then
  timeout 1500 python -m pytest $3 -q -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
  tail -8 gpurun_out/pytest_$TAG.log
fi
timeout 900 python scripts/ab_options.py $OPTS $OPTS > gpurun_out/ab_$TAG.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_$TAG.log
D=gpurun_out/rc_$TAG; mkdir -p $D
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio
python -c "import sys; sys.path.insert(0, '.'); from paper_1509_01149_b200 import build; print(build.source_hash())" > $D/source_hash.txt
timeout 600 python scripts/profile_step.py --config C5 --steps 2 > $D/c5_epi.plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:rollout -s 1 -c 1 --csv --log-file $D/c5_epi.csv \
  python scripts/profile_step.py --config C5 --steps 2 > $D/c5_epi.ncu.log 2>&1
echo "c5_epi C5 4194304 rc=$?" | tee -a $D/manifest.txt
