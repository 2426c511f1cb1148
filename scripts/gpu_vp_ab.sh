# A/B of experiment builds (lib/variants/*) on the config-2 vertex pass only (scripts/vp_bench.py)
for v in default ${VARIANTS:-$(ls paper_2005_07547_b200/lib/variants)}; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  echo "== $v"; timeout 300 python scripts/vp_bench.py --steps ${STEPS:-10} --warmup 3 --streams 2 $VP_ARGS 2>&1 > gpurun_out/vp_$v.log 2>&1; head -${LINES_SHOWN:-3} gpurun_out/vp_$v.log
done
