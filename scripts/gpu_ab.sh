# A/B the default library against experiment builds in lib/variants/* (config-2 vertex pass timing)
for v in default ${VARIANTS:-$(ls paper_2005_07547_b200/lib/variants)}; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  timeout 300 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err || { echo "$v failed"; tail -3 gpurun_out/ab_$v.err; continue; }
  python - "$v" <<'PY'
import json,sys; d=json.loads(open(f'gpurun_out/ab_{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>12s} step {d['ms_per_step']:.3f} ms  vp {d['roofline']['avg_launch_ms']:.3f} ms  {d['value']/1e9:.3f} Gv/s clk {d['clocks']['sm_mhz']}")
PY
done
