# key ncu counters of one steady-state vertex-pass launch per library variant (default + lib/variants/*)
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_branch_resolving.ratio,dram__bytes_read.sum
for v in default ${VARIANTS:-$(ls paper_2005_07547_b200/lib/variants)}; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_vertex_pass_tiled -s 3 -c 1 --csv python scripts/vp_bench.py --steps 1 --warmup 3 --streams 2 > gpurun_out/nq_$v.csv 2>/dev/null
  python - "$v" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/nq_{sys.argv[1]}.csv")) if len(r) > 10]
rows = rows[[r[0] for r in rows].index("ID"):]
h = rows[0]; d = {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows[1:]}
short = lambda k: k.replace("smsp__average_warp_latency_issue_stalled_", "st_").replace(".ratio", "")
print(sys.argv[1], " ".join(f"{short(k).split('.')[0]}={v}" for k, v in d.items()))
PY
done
