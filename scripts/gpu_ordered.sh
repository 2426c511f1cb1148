# ORDERED mode: parity tests, then the config-2 bench line with the per-kernel breakdown
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams.py tests/test_gpu_ordered_scale.py -x -q > gpurun_out/ord_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ord_tests.log
PSTF_ORDERED_DEBUG=1 timeout 300 python bench.py --mode ordered --steps 6 --warmup 8 --no-cpu-baseline > gpurun_out/ord_bench.json 2> gpurun_out/ord_bench.err; echo bench rc=$?
grep "ordered\]" gpurun_out/ord_bench.err | tail -3
python - <<'PY'
import json
d = json.loads(open('gpurun_out/ord_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'])
k = d.get('kernels') or {}
for n, v in sorted(k.items(), key=lambda x: -x[1]['ms_per_step'])[:16]:
    print(f"  {n:40s} {v['ms_per_step']:.3f} ms  x{v['launches']}")
PY
