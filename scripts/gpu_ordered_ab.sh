for v in default noalias; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --mode ordered --steps 6 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']); [print(k, round(v['ms_per_step'],3)) for k, v in list(d['kernels'].items())[:2]]"
done
