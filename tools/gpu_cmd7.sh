# usage: bash tools/gpu_cmd7.sh N — launch list of one int32 sort of N keys (plain run first)
cd $GRAFT_REPO_ROOT
BQ_HOST_LOOP=1 python tools/prof_pass.py --n $1 --passes 0 --sort 2 > gpurun_out/plain7.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv env BQ_HOST_LOOP=1 python tools/prof_pass.py --n $1 --passes 0 --sort 2 > gpurun_out/ncu7.log 2>&1; echo NCU7 $?
