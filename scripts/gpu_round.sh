# One evidence call: the GPU test suite, the per-variant roofline constants (ncu) written to
# profiles/roofline_constants.json on the box (copied to gpurun_out/), then the default bench line
# (which reads them), the bench's ncu launch list and one --set full capture of the C5 step.
#   bash scripts/gpu_round.sh TAG [skip-tests]
TAG=${1:-v}
set -x
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
  tail -15 gpurun_out/pytest_$TAG.log
fi
timeout 1500 bash scripts/gpu_roofline_capture.sh $TAG; echo capture rc=$?
python scripts/roofline_constants.py gpurun_out/rc_$TAG profiles/roofline_constants.json > /dev/null && \
  cp profiles/roofline_constants.json gpurun_out/roofline_constants_$TAG.json; echo constants rc=$?
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-extra --no-latency \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
timeout 900 bash scripts/gpu_ncu_only.sh $TAG
