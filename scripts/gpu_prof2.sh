CMD="python scripts/vp_bench.py --steps 3 --warmup 3 --streams 2"
export PSTF_TILED_CFG=1
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_vertex_pass_tiled|k_ef_blend|k_ef_reduce" -s 9 -c 3 -o gpurun_out/prof2 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu2.log
