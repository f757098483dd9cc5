# one kernel-change iteration: GPU suite, then interleaved A/B of the working build against the
# libraries named on the command line (CUDA-event step and per-kernel times at C5)
TAG=${1:-it}; shift
set -x
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_$TAG.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_$TAG.log
timeout 900 bash scripts/gpu_ab_libs.sh "$@" > gpurun_out/ab_$TAG.txt 2>&1; echo ab rc=$?
cat gpurun_out/ab_$TAG.txt
