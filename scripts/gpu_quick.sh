# quick iteration: selected GPU tests + a short bench (no extras)
TAG=${1:-quick}
SEL=${2:-tests/test_gpu_parity.py}
set -x
timeout 900 python -m pytest $SEL -m gpu -q -x -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-latency --no-cpu-baseline --no-extra > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
cat gpurun_out/bench_$TAG.json
