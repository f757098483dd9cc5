# control-update latency with programmatic (PDL) edges on and off, C1-C3
for c in C1 C2 C3; do
  echo "== $c"; CFG=$c timeout 600 python scripts/ab_latency.py PDL=1 PDL=0 PDL=1 PDL=0
done
