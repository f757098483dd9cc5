set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "warp_specialized" > gpurun_out/ws_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/ws_pytest.log
for K in 65536 131072; do
  CFG=C4 K=$K timeout 300 python scripts/ab_options.py WARP_SPECIALIZED=0 WARP_SPECIALIZED=1 WARP_SPECIALIZED=0 WARP_SPECIALIZED=1
done
