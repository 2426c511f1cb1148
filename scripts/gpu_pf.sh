CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for pf in 0 1 2 3; do echo "== pf $pf"; PSTF_VP_PF=$pf timeout 300 $CMD 2>&1 | sed -n 2p; done
