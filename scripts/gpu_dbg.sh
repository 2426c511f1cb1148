CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for d in 0 32 5 4 1 2 8; do echo "== cfg ${CFG:-1} dbg $d"; PSTF_TILED_CFG=${CFG:-1} PSTF_VP_DBG=$d timeout 300 $CMD 2>&1 | sed -n 2p; done
