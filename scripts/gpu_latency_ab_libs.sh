# control-update latency (graph replay, device p50/p99, host p50) of library builds: default vs exp/*.so
for c in C1 C2 C3 C4; do
  for l in default "$@"; do
    if [ "$l" = default ]; then echo "== $c default"; CFG=$c timeout 600 python scripts/ab_latency.py CUDA_GRAPH=1 CUDA_GRAPH=1;
    else echo "== $c $l"; CFG=$c MPPI_LIB=$PWD/$l timeout 600 python scripts/ab_latency.py CUDA_GRAPH=1 CUDA_GRAPH=1; fi
  done
done
