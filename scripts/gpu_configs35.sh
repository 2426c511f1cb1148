# round-2 documentation lines of configs 3 and 5 (config 5 at its default 2 x L2 capacity and the
# 2^20 eviction stress), as kept in profiles/round2_bench_config*.json
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/c3.json 2> gpurun_out/c3.err; echo c3 rc=$?
timeout 1500 python bench.py --config 5 --no-cpu-baseline > gpurun_out/c5_22.json 2> gpurun_out/c5_22.err; echo c5 rc=$?
timeout 1500 python bench.py --config 5 --capacity-log2 20 --no-cpu-baseline > gpurun_out/c5_20.json 2> gpurun_out/c5_20.err; echo c5_20 rc=$?
for f in c3 c5_22 c5_20; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']/1e9,3),'Gv/s', round(d['ms_per_step'],3),'ms', d['roofline']['kernel'][:60], round(d['roofline']['avg_launch_ms'],3), 'frac', round(d['roofline']['frac'],3))"; done
