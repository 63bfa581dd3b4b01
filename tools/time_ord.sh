cd $GRAFT_REPO_ROOT
for v in main oldord; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  echo "== $v"; BQ_LIB=$L BQ_ORDERED=1 python tools/time_pass.py | tail -1; BQ_LIB=$L python tools/time_rec.py | tail -1
done
