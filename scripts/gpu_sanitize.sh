# compute-sanitizer on small configs of every plant (one tool per gpurun call: $1)
TOOL=${1:-memcheck}
set -x
for c in C1 C3 C4; do
  python scripts/profile_step.py --config $c --K 1024 --steps 2 > gpurun_out/plain_san_$c.log 2>&1 && \
  timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 python scripts/profile_step.py --config $c --K 1024 --steps 2 > gpurun_out/san_${TOOL}_$c.log 2>&1; echo $TOOL $c rc=$?
  tail -3 gpurun_out/san_${TOOL}_$c.log
done
