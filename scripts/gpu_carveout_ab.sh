for c in "1 100" "1 70" "4 0"; do set -- $c
  echo "== cfg $1 carveout $2"; PSTF_TILED_CFG=$1 PSTF_CARVEOUT=$2 timeout 300 python scripts/vp_bench.py --steps 10 --warmup 3 --streams 2 2>&1 | head -2
done
PSTF_TILED_CFG=4 timeout 600 python -m pytest tests/test_gpu_streams.py -x -q -k "crafted" 2>&1 | grep -E "Error|assert|^E " | head -5
