# ncu counters of the endFrame kernels (one-pass vs fused reduce|blend|evict) on config 2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for e in X=1 PSTF_NO_ONEPASS_EF=1; do
  env $e timeout 300 ncu --metrics $M --clock-control none -k regex:"k_ef_" -s 6 -c 3 --csv python scripts/vp_bench.py --steps 2 --warmup 3 --streams 2 > gpurun_out/ef.csv 2>/dev/null
  python - "$e" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open("gpurun_out/ef.csv")) if len(r) > 10]
rows = rows[[r[0] for r in rows].index("ID"):]
h = rows[0]; d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[h.index("Kernel Name")][:22], {})[r[h.index("Metric Name")]] = r[h.index("Metric Value")]
for k, v in d.items():
    print(sys.argv[1], k, " ".join(f"{m.split('.')[0].replace('smsp__average_warp_latency_issue_stalled_','st_')}={x}" for m, x in v.items()))
PY
done
