timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_shard.py -q -m gpu -x 2>&1 | tail -1
for c in 2 3 5 4; do echo "== config $c"; timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1])
print(round(d['value']/1e9,3),'Gv/s', round(d['ms_per_step'],3),'ms', 'vp', round(d['roofline']['avg_launch_ms'],3), 'frac', round(d['roofline']['frac'],3), 'step frac', round(d['step_roofline']['frac'],3), d['field_stats'])
"; done
