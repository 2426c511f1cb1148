# ncu --set full capture of the vertex pass and the fused endFrame (steady state), for profiles/
CMD="python bench.py --steps 3 --warmup 3 --streams 2 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_vertex_pass_tiled|k_ef_fused" -s 6 -c 2 -o gpurun_out/full -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
