CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for v in ${VARIANTS:-1 3 4 5}; do echo "== cfg $v"; PSTF_TILED_CFG=$v timeout 300 $CMD 2>&1 | head -2; done
