cd $GRAFT_REPO_ROOT
for v in main rs5 rs6; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  echo $v; BQ_LIB=$L python tools/time_rec.py
done
