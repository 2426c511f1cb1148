# configs 3/4/5 (documentation runs) + the launch list of the default config-2 bench
for c in 3 5 4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1])
print($c, round(d['value']/1e9,3),'Gv/s', round(d['ms_per_step'],3),'ms', 'vp', round(d['roofline']['avg_launch_ms'],3), 'frac', round(d['roofline']['frac'],3), d['field_stats']['new_keys_last'], d['field_stats']['dropped'])
"; done
LCMD="python bench.py --no-e2e --no-cpu-baseline"
timeout 300 $LCMD > gpurun_out/plain_l.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $LCMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
