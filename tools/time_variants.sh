# usage: bash tools/time_variants.sh v1 v2 ...  (main = the in-tree library)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = main ]; then L=paper_1604_06697_b200/libbq.so; else L=paper_1604_06697_b200/variants/libbq_$v.so; fi
  echo "== $v"; BQ_LIB=$L python tools/time_pass.py | tail -1; BQ_LIB=$L python tools/time_pass.py | tail -1
done
