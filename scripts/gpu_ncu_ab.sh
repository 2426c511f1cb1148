# one ncu --set full capture of the vertex kernel per library variant (VARIANTS="default head ...")
CMD="python bench.py --steps 3 --warmup 3 --streams 2 --no-e2e --no-cpu-baseline"
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset PSTF_LIB_PATH; else export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/$v/libpstf_b200.so; fi
  timeout 300 $CMD > /dev/null 2>&1 || { echo "$v plain run failed"; continue; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vertex_pass_ -s 4 -c 1 -o gpurun_out/ncu_$v -f $CMD > gpurun_out/ncu_$v.log 2>&1; echo "$v ncu rc=$?"
done
