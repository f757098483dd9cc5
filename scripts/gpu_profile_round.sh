# default bench line, its ncu launch list, and one --set full capture of the step (one call)
TAG=${1:-v}
set -x
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-extra \
  > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
timeout 900 bash scripts/gpu_ncu_only.sh $TAG
