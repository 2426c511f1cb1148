# warm-cache DRAM traffic of the endFrame kernels on config 2: single-pass metrics with
# --cache-control none (the kernel runs once, in the application's cache state)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for e in X=1 PSTF_NO_ONEPASS_EF=1; do
  env $e timeout 300 ncu --metrics $M --cache-control none --clock-control none -k regex:"k_ef_|k_vertex" -s 9 -c 3 --csv python scripts/vp_bench.py --steps 2 --warmup 3 --streams 2 > gpurun_out/efw.csv 2>/dev/null
  python - "$e" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open("gpurun_out/efw.csv")) if len(r) > 10]
rows = rows[[r[0] for r in rows].index("ID"):]
h = rows[0]; d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[h.index("ID")] + " " + r[h.index("Kernel Name")][:24], {})[r[h.index("Metric Name")]] = r[h.index("Metric Value")]
for k, v in d.items():
    print(sys.argv[1], k, " ".join(f"{m.split('.')[0]}={x}" for m, x in v.items()))
PY
done
