# config 4 (3840x2160x6 at 2^24) on one GPU, 2 iteration streams (13.7 GB each)
timeout 1500 python bench.py --config 4 --streams 2 --no-cpu-baseline > gpurun_out/c4.json 2> gpurun_out/c4.err; echo rc=$?
tail -c 600 gpurun_out/c4.err
python -c "
import json; d=json.loads(open('gpurun_out/c4.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
