# one ncu --set full capture (with source) of the steady-state vertex pass, for per-line analysis
CMD="python scripts/vp_bench.py --steps 2 --warmup 3 --streams 2"
timeout 300 $CMD > gpurun_out/vp_plain.log 2>&1; echo plain rc=$?; head -3 gpurun_out/vp_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vertex_pass_tiled -s 3 -c 1 -o gpurun_out/vp_src -f $CMD > gpurun_out/ncu_src.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_src.log
