CMD="python scripts/vp_bench.py --steps 3 --warmup 3 --streams 2"
export PSTF_TILED_CFG=${CFG:-2}
timeout 300 $CMD > gpurun_out/plain_cfg.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vertex_pass_tiled -s 3 -c 1 -o gpurun_out/vp_cfg $CMD > gpurun_out/ncu_cfg.log 2>&1; echo ncu rc=$?
