set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
CMD="python bench.py --steps 2 --warmup 2 --streams 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vertex_pass -s 3 -c 1 -o gpurun_out/vp_full $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu2.log
