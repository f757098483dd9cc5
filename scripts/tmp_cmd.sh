for v in "" u2 "" u2; do
  unset MPPI_LIB
  if [ -n "$v" ]; then export MPPI_LIB=$PWD/exp/lib_$v.so; fi
  echo "variant $v"; timeout 300 python scripts/ab_options.py FUSED_NOISE=1
done
