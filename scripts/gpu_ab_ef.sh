# A/B of endFrame variants (lib/variants/*): step time and the fused endFrame kernel per step
for v in default ${VARIANTS:-$(ls paper_2005_07547_b200/lib/variants)}; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  timeout 300 python bench.py --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abef_$v.json 2>gpurun_out/abef_$v.err || { echo "$v failed"; continue; }
  python - "$v" <<'PY'
import json,sys; d=json.loads(open(f'gpurun_out/abef_{sys.argv[1]}.json').read().strip().splitlines()[-1])
k=d['kernels'].get('k_ef_fused',{}).get('ms_per_step',0)
print(f"{sys.argv[1]:>8s} step {d['ms_per_step']:.3f} ms  ef {k:.4f} ms  {d['value']/1e9:.3f} Gv/s")
PY
done
