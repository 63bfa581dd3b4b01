# usage: bash tools/gpu_cmd17.sh V1 V2 ... — multiway parity subset, then c3/c5 and c2 (ways 8) timing per variant
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keyidx.py -q -m gpu -x -k "multiway or mw or ways or keyidx or pair or nan or f64" 2>&1 | tail -3
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  BQ_LIB=$L timeout 300 python tools/time_configs.py --configs c3,c5 2>&1 | grep -v "ascending\|descending\|swapped" | sed "s/^/$v /" | cut -c1-120
done
