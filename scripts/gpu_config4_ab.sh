# config 4: the hot-slot variant chosen automatically against forced off / on
for e in auto 0 1; do
  if [ "$e" = auto ]; then unset PSTF_RED_AGG; else export PSTF_RED_AGG=$e; fi
  timeout 1500 python bench.py --config 4 --streams 2 --steps 6 --no-cpu-baseline --no-e2e > gpurun_out/c4_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c4_$e.json').read().strip().splitlines()[-1])
print('$e', d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'])"
done
