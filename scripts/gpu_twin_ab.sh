for r in 1 2; do
for v in default twin2 twin2on; do
  case $v in default) unset PSTF_LIB_PATH; unset PSTF_TWIN_FORCE;; twin2) export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/twin2/libpstf_b200.so; unset PSTF_TWIN_FORCE;; twin2on) export PSTF_LIB_PATH=$PWD/paper_2005_07547_b200/lib/variants/twin2/libpstf_b200.so; export PSTF_TWIN_FORCE=1;; esac
  echo "== $v"; timeout 300 python scripts/vp_bench.py --steps 10 --warmup 3 --streams 2 2>&1 | head -2
done; done
