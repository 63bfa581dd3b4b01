# usage: bash tools/gpu_mw8t.sh — TMA-staged 8-way scatter: parity, then c1/c2/c3/c5 by ways, new vs old scatter
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multiway or keyidx or full" 2>&1 | tail -5
for v in main old; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  for w in 2 8 16; do BQ_LIB=$L timeout 300 python tools/time_configs.py --configs c1,c2 --ways $w 2>&1 | sed "s/^/$v w$w /" | cut -c1-160; done
  BQ_LIB=$L timeout 300 python tools/time_configs.py --configs c3,c5 2>&1 | sed "s/^/$v w0 /" | cut -c1-160
done
