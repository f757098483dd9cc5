# round-2 parity batch: the new oracle-anchored GPU tests, then a pipe-split ncu capture of C5
set -x
timeout 1500 python -m pytest tests/test_gpu_bm32_exhaustive.py tests/test_gpu_general_sigma.py \
  tests/test_gpu_c5_full.py tests/test_gpu_closed_loop.py tests/test_gpu_parity.py -q -s -rf \
  > gpurun_out/r2a_pytest.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/r2a_pytest.log
timeout 900 bash scripts/gpu_ncu_only.sh ${1:-r2a}
