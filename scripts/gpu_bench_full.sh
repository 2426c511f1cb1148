# full bench + launch list + ncu --set full capture of the dominant kernel (for profiles/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err
# launch list of the bench's own default step sequence (summarise with --skip-steps 3)
LCMD="python bench.py --no-e2e --no-cpu-baseline"
timeout 300 $LCMD > gpurun_out/plain_l.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $LCMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
CMD="python bench.py --steps 3 --warmup 3 --streams 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_vertex_pass_tiled|k_ef_fused" -s 6 -c 2 -o gpurun_out/full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
