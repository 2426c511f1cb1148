# parity tests, then the bench, then a kernel launch list (ncu) of a short bench
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -5 gpurun_out/bench.err
