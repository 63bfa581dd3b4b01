# usage: bash tools/gpu_cmd20.sh — c1-sized int32 sorts by ways and kernel family (small-n policy)
cd $GRAFT_REPO_ROOT
for v in main old; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  for w in 2 8 16; do BQ_LIB=$L python tools/time_configs.py --configs c1 --ways $w 2>&1 | sed "s/^/$v w$w /" | cut -c1-120; done
done
SWEEP_KINDS=i32 SWEEP_LOGS=16,18,20,22,24 python tools/ways_sweep.py 2>&1 | tail -8
