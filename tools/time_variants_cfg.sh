# usage: bash tools/time_variants_cfg.sh CONFIGS v1 v2 ...  (main = the in-tree library): time_configs per variant
cd $GRAFT_REPO_ROOT
C=$1; shift
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  BQ_LIB=$L timeout 300 python tools/time_configs.py --configs $C 2>&1 | sed "s/^/$v /" | cut -c1-150
done
