# usage: bash tools/gpu_var.sh V1 V2 ... — c1/c2/c3/c5 timing per library variant (main = the in-tree build)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  BQ_LIB=$L timeout 300 python tools/time_configs.py --configs ${CFGS:-c1,c2,c3,c5} 2>&1 | sed "s/^/$v /" | cut -c1-100
done
