set -x
CMD="python scripts/vp_bench.py --steps 4 --warmup 3 --streams 2"
timeout 300 $CMD > gpurun_out/vp_tma.log 2>&1; echo rc=$?; cat gpurun_out/vp_tma.log | head -12
PSTF_NO_TMA=1 timeout 300 $CMD > gpurun_out/vp_notma.log 2>&1; echo rc=$?; head -4 gpurun_out/vp_notma.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vertex_pass_tiled -s 3 -c 1 -o gpurun_out/vp_tiled $CMD > gpurun_out/ncu_tiled.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_tiled.log
