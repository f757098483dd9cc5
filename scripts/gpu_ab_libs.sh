# A/B of library builds (kernel-variant experiments): the default build and exp/*.so, interleaved
# bash scripts/gpu_ab_libs.sh exp/lib_a.so exp/lib_b.so ...
for rep in 1 2; do
  echo "== default"; timeout 300 python scripts/ab_options.py FUSED_REDUCTION=1
  for l in "$@"; do echo "== $l"; MPPI_LIB=$PWD/$l timeout 300 python scripts/ab_options.py FUSED_REDUCTION=1; done
done
