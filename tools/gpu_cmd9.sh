# usage: bash tools/gpu_cmd9.sh WAYS REGEX SKIP TAG — ncu --set full of one launch of REGEX in one int32 c2 sort with WAYS
cd $GRAFT_REPO_ROOT
BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --ways $1 > gpurun_out/plain9.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s ${3:-0} -c 1 -o gpurun_out/prof_$4 env BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --ways $1 > gpurun_out/ncu9.log 2>&1; echo NCU9 $?
