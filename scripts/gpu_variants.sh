CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for v in 0 1 2; do echo "== tiled cfg $v"; PSTF_TILED_CFG=$v timeout 300 $CMD 2>&1 | head -3; done
echo "== no tma"; PSTF_NO_TMA=1 timeout 300 $CMD 2>&1 | head -3
