# Round-2 measurement pass (all into gpurun_out/r2_*): the bench lines of profiles/round2_*,
# the launch list and one ncu --set full capture of the dominant kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo ref rc=$?
timeout 600 python bench.py --mode ordered --no-cpu-baseline > gpurun_out/r2_ordered.json 2> gpurun_out/r2_ordered.err; echo ordered rc=$?
timeout 600 python bench.py --force-sharded --no-cpu-baseline > gpurun_out/r2_sharded.json 2> gpurun_out/r2_sharded.err; echo sharded rc=$?
LCMD="python bench.py --no-e2e --no-cpu-baseline"
timeout 300 $LCMD > gpurun_out/r2_plain_l.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $LCMD > gpurun_out/r2_ncu_launch.log 2>&1; echo ncu1 rc=$?
CMD="python bench.py --steps 3 --warmup 3 --streams 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/r2_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_vertex_pass_tiled|k_ef_onepass|k_ef_tail" -s 9 -c 3 -o gpurun_out/r2_full $CMD > gpurun_out/r2_ncu_full.log 2>&1; echo ncu2 rc=$?
tail -2 gpurun_out/r2_ncu_full.log
