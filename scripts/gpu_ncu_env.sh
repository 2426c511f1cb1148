# key ncu counters of one steady-state vertex-pass launch for each environment setting in $ENVS
# (e.g. ENVS="PSTF_VP_WARP=0 PSTF_VP_WARP=1"); kernel regex $KRE (default: any vertex pass)
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_branch_resolving.ratio,smsp__average_warp_latency_issue_stalled_sleeping.ratio,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
for e in ${ENVS:-X=1}; do
  env $e timeout 300 ncu --metrics $M --clock-control none -k regex:${KRE:-k_vertex_pass} -s 3 -c 1 --csv python scripts/vp_bench.py --steps 1 --warmup 3 --streams 2 > gpurun_out/ne.csv 2>/dev/null
  python - "$e" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/ne.csv")) if len(r) > 10]
rows = rows[[r[0] for r in rows].index("ID"):]
h = rows[0]; d = {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows[1:]}
short = lambda k: k.replace("smsp__average_warp_latency_issue_stalled_", "st_").replace(".ratio", "")
print(sys.argv[1], rows[1][h.index("Kernel Name")][:30], " ".join(f"{short(k).split('.')[0]}={v}" for k, v in d.items()))
PY
done
