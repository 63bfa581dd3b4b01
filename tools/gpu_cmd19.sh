# usage: bash tools/gpu_cmd19.sh V... — DRAM bytes and time of the records gather per variant (ncu), then c5 timing
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  BQ_LIB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:gather python tools/one_sort.py c5 2>/dev/null | grep -i "gather" | tail -3 | sed "s/^/$v /" | cut -c1-40,100-300
done
unset BQ_HOST_LOOP
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  BQ_LIB=$L timeout 300 python tools/time_configs.py --configs c5 2>&1 | sed "s/^/$v /" | cut -c1-120
done
