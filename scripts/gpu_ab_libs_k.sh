# A/B of library builds at several K (C5 plant/forest): bash scripts/gpu_ab_libs_k.sh "K1 K2 ..." exp/lib_a.so ...
KS=$1; shift
for K in $KS; do
  for rep in 1 2; do
    echo "== K=$K default"; K=$K timeout 300 python scripts/ab_options.py FUSED_REDUCTION=1
    for l in "$@"; do echo "== K=$K $l"; K=$K MPPI_LIB=$PWD/$l timeout 300 python scripts/ab_options.py FUSED_REDUCTION=1; done
  done
done
