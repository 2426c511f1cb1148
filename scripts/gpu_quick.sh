# parity + golden GPU tests, then a short config-2 bench (no e2e / cpu legs); one-line summary
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python - <<'PY'
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
k=d['kernels']; top=sorted(k.items(), key=lambda kv:-kv[1]['ms_per_step'])[:5]
print(round(d['value']/1e9,3),'Gv/s step', round(d['ms_per_step'],3),'ms vp', round(d['roofline']['avg_launch_ms'],3), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
print([(n[:28], round(v['ms_per_step'],4)) for n,v in top])
PY
done
