# Per-sample-step roofline numerators of every rollout variant the bench reports (FP32 FLOP
# counters, warp instructions, DRAM bytes), one ncu capture each of the second step's rollout,
# tagged with the source hash of the tree that ran.  Then, on the CPU:
#   python scripts/roofline_constants.py gpurun_out/rc_<TAG>   -> profiles/roofline_constants.json
TAG=${1:-rc}
D=gpurun_out/rc_$TAG
mkdir -p $D
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active
python -c "import sys; sys.path.insert(0, '.'); from paper_1509_01149_b200 import build; print(build.source_hash())" > $D/source_hash.txt
git rev-parse HEAD > $D/git_head.txt 2>/dev/null || true
run() {   # name config K [env]
  name=$1; cfg=$2; K=$3; shift 3
  env "$@" timeout 600 python scripts/profile_step.py --config $cfg --K $K --steps 2 > $D/$name.plain.log 2>&1 && \
  env "$@" timeout 900 ncu --metrics $M --clock-control none -k regex:rollout -s 1 -c 1 --csv \
      --log-file $D/$name.csv python scripts/profile_step.py --config $cfg --K $K --steps 2 > $D/$name.ncu.log 2>&1
  echo "$name $cfg $K $* rc=$?" | tee -a $D/manifest.txt
}
run c5_epi C5 4194304
run c5_sep C5 4194304 MPPI_OPTS=FUSED_REDUCTION=0
run c5_ctg C5 4194304 CTG=1
run c4_k65536 C4 65536
run c4_k4096 C4 4096
run c3 C3 16384
run c2 C2 4096
run c1 C1 256
run c1_k1000 C1 1000
ls -la $D
