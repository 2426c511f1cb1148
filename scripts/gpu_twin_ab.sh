# twin Lo/LoE stores on config 2: the TWIN instantiation (default for fresh store pairs)
# against separate probes (PSTF_NO_TWIN=1), interleaved twice
for r in 1 2; do
  for v in twin separate; do
    if [ "$v" = separate ]; then export PSTF_NO_TWIN=1; else unset PSTF_NO_TWIN; fi
    echo "== $v"; timeout 300 python scripts/vp_bench.py --steps 10 --warmup 3 --streams 2 2>&1 | head -2
  done
done
