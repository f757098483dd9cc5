timeout 300 python scripts/ab_options.py OBSTACLE_GRID=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf 2>&1 | tail -3
