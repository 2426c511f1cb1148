timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gpu_tests.log
CMD="python scripts/vp_bench.py --steps 6 --warmup 3 --streams 3"
for v in 1 0 2; do echo "== tiled cfg $v"; PSTF_TILED_CFG=$v timeout 300 $CMD 2>&1 | head -7; done
