# usage: bash tools/gpu_cmd4.sh — launch lists of one c3 (f64 2^27) and one c5 (records 2^26) sort
cd $GRAFT_REPO_ROOT
for k in f64:134217728 rec:67108864; do
  kind=${k%%:*}; n=${k##*:}
  python tools/prof_pass.py --kind $kind --n $n --passes 0 --sort 1 > gpurun_out/plain_$kind.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$kind.csv python tools/prof_pass.py --kind $kind --n $n --passes 0 --sort 1 > gpurun_out/ncu_$kind.log 2>&1; echo NCU $kind $?
done
