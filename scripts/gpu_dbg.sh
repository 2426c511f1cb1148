CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for d in 0 1 2 3 4 5 32; do echo "== dbg $d"; PSTF_VP_DBG=$d timeout 300 $CMD 2>&1 | sed -n 2p; done
